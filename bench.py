#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W]
                    [--workload cfg5|cfg2|cfg1|cfg3|cfg4] [--impl ours|reference]

Default workload: BASELINE config 5, the sharded config the headline metric is
quoted on -- 4,096 sources x 60 s at 48 kHz (47 GB fp32), each at one of 1,250
directions (K 100, nnz 24), per-ear f of 101 taps, summed to a stereo mix.
``--gpus N`` runs one process per GPU: under torchrun it reads
RANK/WORLD_SIZE; without a launcher it re-executes itself under
``torch.distributed.run`` with N processes.  Sources are partitioned by
direction (dist.MixShard), every rank renders its partial mix on the tensor
cores (k_mix_mma), one NCCL reduce sums the partials onto rank 0, which applies
f.  Metric: output samples/s counted as src x ear (each source has one
direction), whole job, max over ranks.  At N = 1 the line also carries
``fused_render``: config 2 (one source through 1,250 directions x 2 ears in one
fused f->g launch), the north_star's "fused kernel >= 60% of roofline" bar.

``value``     : device-resident throughput, CUDA events around each step on
                the launching stream, L2 flushed (256 MiB write) between steps,
                max over ranks.
``e2e``       : same metric through the public API with host buffers: pinned
                host -> device copy of the step's inputs, the render, device ->
                host copy of the result, per step.
``roofline``  : dominant kernel's algorithmic bytes / its event-timed duration
                vs MEASURED_PEAKS.json.
``cpu_baseline`` / ``--impl reference``: the reference's own compiled CPU
                kernels (oracle/_ref, built from pkg/src/toepnmf/engine/_kernels.pyx)
                composed as Renderer.render does, on all host cores, on a
                bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# --------------------------------------------------------------- helpers ----


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured", "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0))}
    except Exception:
        return {"hbm_gbs": 6650.0, "src": "fallback", "sm_max_mhz": 1965.0}


FP32_LANES_PER_SM = 128


def _traffic(workload):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)[workload]
        return {"bytes_per_launch": t["dram_bytes_read"] + t["dram_bytes_write"], "source": t["source"]}
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    NAMES = {
        "nvmlClocksEventReasonGpuIdle": "gpu_idle",
        "nvmlClocksEventReasonApplicationsClocksSetting": "applications_clocks_setting",
        "nvmlClocksEventReasonSwPowerCap": "sw_power_cap",
        "nvmlClocksEventReasonHwSlowdown": "hw_slowdown",
        "nvmlClocksEventReasonSyncBoost": "sync_boost",
        "nvmlClocksEventReasonSwThermalSlowdown": "sw_thermal_slowdown",
        "nvmlClocksEventReasonHwThermalSlowdown": "hw_thermal_slowdown",
        "nvmlClocksEventReasonHwPowerBrakeSlowdown": "hw_power_brake_slowdown",
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples = []
        self.reasons = 0
        self.ok = False
        self._stop = threading.Event()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            uuid = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            except Exception:
                pass
            self.h = None
            if uuid:
                for i in range(pynvml.nvmlDeviceGetCount()):
                    h = pynvml.nvmlDeviceGetHandleByIndex(i)
                    u = pynvml.nvmlDeviceGetUUID(h)
                    u = u.decode() if isinstance(u, bytes) else u
                    if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                        self.h = h
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.sm_max = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": ["unavailable"]}
        names = []
        for attr, name in self.NAMES.items():
            bit = getattr(self.nv, attr, None)
            if bit is not None and self.reasons & bit:
                names.append(name)
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.sm_max),
                "reasons": names, "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def timed(step, K: int, W: int, world: int, flush=None, stream=None):
    """W warm-ups, then K steps each bracketed by CUDA events on `stream`;
    L2 flushed between steps (outside the events).  Returns per-step ms."""
    import torch
    s = stream or torch.cuda.current_stream()
    for _ in range(W):
        step()
        if flush:
            flush()
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    wall0 = time.perf_counter()
    for i in range(K):
        if flush:
            flush()
        evs[i][0].record(s)
        step()
        evs[i][1].record(s)
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    return [a.elapsed_time(b) for a, b in evs], wall


# ------------------------------------------------------ reference (CPU) ----

_REF_STATE = {}


def _ref_worker_init(payload):
    import oracle
    mod = oracle.ref_kernels()
    kind = "reference"
    if mod is None:  # reference not built here: fall back to the C restatement
        mod = oracle
        kind = "port"
    _REF_STATE.update(payload)
    _REF_STATE["mod"] = mod
    _REF_STATE["kind"] = kind
    _REF_STATE["yf"] = {}


def _ref_render_rows(task):
    """Renderer.render composition on CPU: y*f cached per ear, conv_sparse per row."""
    ear, rows = task
    st = _REF_STATE
    mod = st["mod"]
    if ear not in st["yf"]:
        st["yf"][ear] = mod.conv_dense(st["y"], st["f"][ear])[0]
    yf = st["yf"][ear]
    n = 0
    for r in rows:
        idx, vals = st["rows"][r]
        out, _ = mod.conv_sparse(yf, idx, vals, st["K"])
        n += out.size
    return n


def _ref_worker_init_cfg3(payload):
    """cfg3 workers: y*f of every (point, ear) rendered up front in the parent
    (shared by fork) -- the reference renders it once per renderer and reuses
    it for all 1,250 directions (< 3% of a point's work)."""
    _ref_worker_init(payload)
    _REF_STATE["yf"] = dict(payload["yf"])


def _ref_render_point_rows(task):
    """cfg3 sweep: the Renderer.render composition for rows of one sweep point."""
    p, ear, rows = task
    st = _REF_STATE
    mod = st["mod"]
    pt = st["pts"][p]
    if (p, ear) not in st["yf"]:
        st["yf"][(p, ear)] = mod.conv_dense(st["y"], pt["f"][ear])[0]
    yf = st["yf"][(p, ear)]
    n = 0
    for r in rows:
        idx, vals = pt["rows"][r]
        out, _ = mod.conv_sparse(yf, idx, vals, pt["K"])
        n += out.size
    return n


def _ref_mix_sources(task):
    """Per-source Renderer.render for both ears, accumulated in fp64 (mixdown configs)."""
    st = _REF_STATE
    mod = st["mod"]
    acc = {}
    n = 0
    for s in task:
        y = st["ysrc"][s]
        for e in range(st["ears"]):
            yf = mod.conv_dense(y, st["f"][e])[0]
            idx, vals = st["rows"][e * st["dirs"] + st["src_dir"][s]]
            out, _ = mod.conv_sparse(yf, idx, vals, st["K"])
            acc[e] = out if e not in acc else acc[e] + out
            n += out.size
    return n


def _single_core_rate(payload, fn, tasks, budget_s):
    """The same reference work in this process on one core: samples/s over ~budget_s."""
    _ref_worker_init(payload)
    n, i = 0, 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < budget_s and i < len(tasks):
        n += fn(tasks[i])
        i += 1
    return n / (time.perf_counter() - t0)


def reference_step_factory(workload: str, cores: int):
    """Returns (step_fn -> samples computed, description, kind, pool, single_core_rate_fn)."""
    import multiprocessing as mp

    from paper_1502_03162_b200 import synth
    from paper_1502_03162_b200.batch import model_rows

    if workload in ("cfg1", "cfg2"):
        cfg = synth.CONFIGS[workload]
        ms = synth.models(cfg, seed=2)
        y = synth.source(cfg.ny, seed=22)
        rows = model_rows(ms)
        payload = {"y": y, "f": [m.resonance_taps for m in ms], "rows": rows, "K": cfg.K}
        ctx = mp.get_context("fork")
        pool = ctx.Pool(cores, initializer=_ref_worker_init, initargs=(payload,))
        per_ear = cfg.dirs
        chunk = max(1, per_ear // max(1, cores // cfg.ears) // 4)
        tasks = [(e, list(range(e * per_ear + d, e * per_ear + min(per_ear, d + chunk))))
                 for e in range(cfg.ears) for d in range(0, per_ear, chunk)]

        def step():
            return sum(pool.map(_ref_render_rows, tasks, chunksize=1))

        def single(budget_s=3.0):
            return _single_core_rate(payload, _ref_render_rows, tasks, budget_s)

        desc = "full %s per step: %d channels x %d samples, Renderer.render composition" % (
            workload, cfg.ears * cfg.dirs, cfg.ny + cfg.M - 1)
        kind = "reference" if _probe_ref() else "port"
        return step, desc, kind, pool, single
    if workload == "cfg3":
        # every sweep point, bounded: 4 x cores directions of each ear over the
        # full 441,000-sample source (the reference's per-row cost does not
        # depend on which directions); per-point rates kept on step.rates
        pts = synth.cfg3_points()
        y = synth.source(pts[0].ny, seed=3)
        payload = {"y": y, "pts": []}
        for cfg in pts:
            ms = synth.models(cfg, seed=cfg.K * 1000 + cfg.nnz)
            payload["pts"].append({"f": [m.resonance_taps for m in ms], "rows": model_rows(ms), "K": cfg.K})
        import oracle
        mod = oracle.ref_kernels() or oracle
        payload["yf"] = {(p, e): mod.conv_dense(y, f)[0] for p, pt in enumerate(payload["pts"])
                         for e, f in enumerate(pt["f"])}
        ctx = mp.get_context("fork")
        pool = ctx.Pool(cores, initializer=_ref_worker_init_cfg3, initargs=(payload,))
        nd = min(pts[0].dirs, max(8, 4 * cores))
        tasks = [[(p, e, list(range(e * cfg.dirs + d, e * cfg.dirs + min(nd, d + 4))))
                  for e in range(cfg.ears) for d in range(0, nd, 4)] for p, cfg in enumerate(pts)]

        def step():
            n = 0
            for p, cfg in enumerate(pts):
                t0 = time.perf_counter()
                k = sum(pool.map(_ref_render_point_rows, tasks[p], chunksize=1))
                dt = time.perf_counter() - t0
                r = step.rates.setdefault(cfg.name, [0, 0.0])
                r[0] += k
                r[1] += dt
                n += k
            return n
        step.rates = {}

        def single(budget_s=3.0):
            # one core: the nnz-16 point at K 100 (cfg2's sparsity), its y*f precomputed
            p = [c.name for c in pts].index("cfg3_K100_nnz16")
            _ref_worker_init_cfg3(payload)
            n, i = 0, 0
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < budget_s and i < len(tasks[p]):
                n += _ref_render_point_rows(tasks[p][i])
                i += 1
            return n / (time.perf_counter() - t0)

        desc = ("17 cfg3 points per step, each %d directions x 2 ears x %d samples (full source), "
                "Renderer.render composition (y*f per ear rendered once, before timing)"
                % (nd, pts[0].ny + pts[0].M - 1))
        kind = "reference" if _probe_ref() else "port"
        return step, desc, kind, pool, single
    if workload in ("cfg4", "cfg5"):
        cfg = synth.CONFIGS[workload]
        ms = synth.models(cfg, seed=5)
        sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
        # bounded sample: 2 s of audio for `cores` sources per step
        T = 2 * synth.FS_48K
        nsrc = min(cfg.sources, max(cores, 16))
        rng = np.random.default_rng(0)
        ysrc = [rng.standard_normal(T).astype(np.float32).astype(np.float64) for _ in range(nsrc)]
        payload = {"ysrc": ysrc, "f": [m.resonance_taps for m in ms], "rows": model_rows(ms), "K": cfg.K,
                   "ears": cfg.ears, "dirs": cfg.dirs, "src_dir": sd[:nsrc]}
        ctx = mp.get_context("fork")
        pool = ctx.Pool(cores, initializer=_ref_worker_init, initargs=(payload,))
        tasks = [[s] for s in range(nsrc)]

        def step():
            # src x ear samples of the bounded sample (output T + M - 1 per source-ear)
            return sum(pool.map(_ref_mix_sources, tasks, chunksize=1))

        def single(budget_s=3.0):
            return _single_core_rate(payload, _ref_mix_sources, tasks, budget_s)

        desc = "%d sources x 2 s (%d samples) per step, %s laws; per-source Renderer.render + fp64 sum" % (
            nsrc, T, workload)
        kind = "reference" if _probe_ref() else "port"
        return step, desc, kind, pool, single
    raise SystemExit("no reference arm for workload %s" % workload)


def _probe_ref():
    import oracle
    return oracle.ref_kernels() is not None


def _ref_stream_blocks(task):
    """Streaming reference: per 256-sample block and
    source, Renderer.render over [199-sample history | block] with the
    reference's kernels; the block's outputs are samples [199, 199 + B) of that
    window render (exact), summed over sources in fp64."""
    st = _REF_STATE
    mod = st["mod"]
    b, srcs = task
    B, H = st["B"], st["H"]
    n = 0
    acc = np.zeros((st["ears"], B))
    for s in srcs:
        y = st["ysrc"][s]
        lo = b * B - H
        win = y[max(0, lo):(b + 1) * B]
        if lo < 0:
            win = np.concatenate([np.zeros(-lo), win])
        for e in range(st["ears"]):
            yf = mod.conv_dense(win, st["f"][e])[0]
            idx, vals = st["rows"][e * st["dirs"] + st["src_dir"][s]]
            out, _ = mod.conv_sparse(yf, idx, vals, st["K"])
            acc[e] += out[H:H + B]
            n += B
    return n


def reference_stream_factory(cores: int):
    """cfg4 CPU baseline: reference calls per block over a 199-sample history window."""
    import multiprocessing as mp

    from paper_1502_03162_b200 import synth
    from paper_1502_03162_b200.batch import model_rows

    cfg = synth.CONFIGS["cfg4"]
    ms = synth.models(cfg, seed=4)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
    nblk = 8  # bounded sample: 8 consecutive blocks of all 512 sources per step
    T = (nblk + 1) * cfg.block
    rng = np.random.default_rng(0)
    ysrc = [rng.standard_normal(T).astype(np.float32).astype(np.float64) for _ in range(cfg.sources)]
    payload = {"ysrc": ysrc, "f": [m.resonance_taps for m in ms], "rows": model_rows(ms), "K": cfg.K,
               "ears": cfg.ears, "dirs": cfg.dirs, "src_dir": sd, "B": cfg.block, "H": cfg.M - 1}
    ctx = mp.get_context("fork")
    pool = ctx.Pool(cores, initializer=_ref_worker_init, initargs=(payload,))
    per = max(1, cfg.sources // cores)
    tasks = [(b, list(range(s, min(cfg.sources, s + per)))) for b in range(1, nblk + 1)
             for s in range(0, cfg.sources, per)]

    def step():
        return sum(pool.map(_ref_stream_blocks, tasks, chunksize=1))

    def single(budget_s=3.0):
        return _single_core_rate(payload, _ref_stream_blocks, tasks, budget_s)

    desc = ("%d blocks x %d sources x 2 ears per step: per block and source, Renderer.render over the "
            "199-sample history + 256-sample block (reference kernels), outputs [199, 455) summed in fp64"
            % (nblk, cfg.sources))
    kind = "reference" if _probe_ref() else "port"
    return step, desc, kind, pool, single


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_factory(wl, cores):
    if wl == "cfg4":
        return reference_stream_factory(cores)
    return reference_step_factory(wl, cores)


METRIC = "output samples/s (src x dir x ear)"


def workload_config(wl: str, world: int) -> dict:
    """The config dict both arms print for a workload (identical keys and values)."""
    from paper_1502_03162_b200 import synth
    if wl == "cfg3":
        return {"workload": "cfg3", "sources": 1, "directions": 1250, "ears": 2, "signal_len": 441_000,
                "K": [50, 100, 150], "nnz": [4, 8, 16, 32, 64, "K"], "points": 17,
                "parallelism": "one GPU per point", "l2": "flushed between steps (256 MiB write)"}
    cfg = synth.CONFIGS[wl]
    d = {"workload": wl, "sources": cfg.sources, "directions": cfg.dirs, "ears": cfg.ears, "signal_len": cfg.ny,
         "K": cfg.K, "Lf": cfg.lf, "nnz": cfg.nnz}
    if wl in ("cfg1", "cfg2"):
        d["out_len"] = cfg.ny + cfg.M - 1
        d["parallelism"] = "independent sources x %d (one per GPU), no collective" % world
        d["l2"] = "flushed between steps (256 MiB write)"
    elif wl == "cfg4":
        d["block"] = cfg.block
        d["parallelism"] = "one stream per GPU (replicas), no collective"
        d["l2"] = "stream state resident; inputs 5.9 GB > L2"
    else:
        d["parallelism"] = "sources by direction over %d GPU(s), one NCCL reduce of the stereo partial" % world
        d["l2"] = "inputs (47 GB) larger than L2; 256 MiB write between steps"
    return d


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    wl = args.workload
    step, desc, kind, pool, _ = _ref_factory(wl, cores)
    try:
        for _ in range(args.warmup):
            step()
        times, counts = [], []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            counts.append(step())
            times.append(time.perf_counter() - t0)
    finally:
        pool.close()
        pool.join()
    total = sum(times)
    value = sum(counts) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if wl == "cfg5" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE laws)",
        "config": workload_config(wl, args.gpus),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind, "sample": desc,
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if getattr(step, "rates", None):
        line["cpu_baseline"]["points"] = {k: n / t for k, (n, t) in step.rates.items()}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_line(workload):
    cores = os.cpu_count() or 1
    step, desc, kind, pool, single = _ref_factory(workload, cores)
    # repeat the bounded sample until ~10 s of CPU work has been timed
    try:
        step()  # warm
        n, reps = 0, 0
        t0 = time.perf_counter()
        while True:
            n += step()
            reps += 1
            dt = time.perf_counter() - t0
            if dt >= 10.0 or reps >= 1000:
                break
    finally:
        pool.close()
        pool.join()
    out = {"value": n / dt, "unit": "samples/s", "cores": cores, "kind": kind,
           "sample": "%s; %d repetitions" % (desc, reps), "seconds": dt,
           "single_core_value": single(3.0), "cpu_model": _cpu_model()}
    if getattr(step, "rates", None):
        out["points"] = {k: m / t for k, (m, t) in step.rates.items()}
    return out


# ------------------------------------------------------------ our arm ------


def _flush_fn():
    import torch
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def flush():
        buf.fill_(0.0)
    return flush


def bench_render(args, world, rank, local, workload="cfg2", steps=None, warmup=None, e2e=True):
    """cfg1/cfg2: one source through every (ear, direction), fused f->g (k_render_mma)."""
    import torch

    from paper_1502_03162_b200 import batch, synth

    steps = steps or args.steps
    warmup = warmup or args.warmup
    cfg = synth.CONFIGS[workload]
    ms = synth.models(cfg, seed=2)
    # N GPUs: weak scaling over independent sources -- rank r renders its own
    # source (seed 22 + r) through every (ear, direction) (no collective)
    y_host = synth.source(cfg.ny, seed=22 + rank).astype(np.float32)
    y = torch.from_numpy(y_host).cuda()
    br = batch.BatchRenderer(ms)
    out = br.alloc(y.numel())
    L = br.out_len(cfg.ny)
    br.render_all(y, out=out)  # validates inputs once (finite check) and builds device state
    samples_local = br.ears * br.dirs * L
    samples_global = samples_local * world
    flush = _flush_fn()

    def step():
        br.render_all(y, out=out, check_finite=False)

    with ClockSampler(local) as clk:
        ms_steps, wall = timed(step, steps, warmup, world, flush)
    tot_ms = sum(ms_steps)
    tot_ms_max = _max_over_ranks(tot_ms, world)
    value = samples_global * steps / (tot_ms_max * 1e-3)
    kern_ms = statistics.mean(ms_steps)
    peaks = _peaks()
    alg_bytes = samples_local * 4 + y.numel() * 4 + int(br.row_nnz.sum()) * 8 + cfg.ears * cfg.lf * 4
    achieved_gbs = alg_bytes / (kern_ms * 1e-3) / 1e9
    flops = (2.0 * int(br.row_nnz.sum()) * (y.numel() + cfg.lf - 1) + 2.0 * cfg.ears * cfg.lf * (y.numel() + br.M))
    roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved_gbs / peaks["hbm_gbs"], "traffic": _traffic(workload),
            "peak_src": peaks["src"],
            "kernel": {"tensor": "k_render_mma (tcgen05.mma split-fp16, TMA-multicast G; 6-CTA clusters + a concurrent "
                                 "2-CTA-cluster launch on the SMs they leave idle)",
                       "window": "k_render<112,true,16> (TMEM window + FFMA2)",
                       "banded": "k_sparse_generic"}[br.native.path()],
            "kernel_ms": kern_ms, "fp32_tflops": flops / (kern_ms * 1e-3) / 1e12,
            "alg_bytes_per_launch": alg_bytes}
    e2e_obj = None
    if e2e and not args.no_e2e:
        y_pin = torch.from_numpy(y_host).pin_memory()
        out_pin = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        e2e_steps = max(2, min(steps, 5))

        def e2e_step():
            y.copy_(y_pin, non_blocking=True)
            r = br.render_all(y, out=out)  # the user's call: includes the fused non-finite check
            out_pin.copy_(out, non_blocking=True)
            return r

        ms_e2e, _ = timed(e2e_step, e2e_steps, 1, world)
        e2e_ms = _max_over_ranks(sum(ms_e2e), world)
        e2e_obj = {"value": samples_global * e2e_steps / (e2e_ms * 1e-3), "unit": "samples/s",
                   "h2d_bytes_per_step": int(y_pin.numel() * 4), "d2h_bytes_per_step": int(out_pin.numel() * 4),
                   "ms_per_step": e2e_ms / e2e_steps}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": tot_ms_max / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded: y~N(0,1), f decaying Gaussian, g half-normal at uniform positions)",
        "config": workload_config(workload, world),
        "roofline": roof, "e2e": e2e_obj, "gpu_launches": steps * br.native.kernels(cfg.ny),
        "clocks": clk.summary(),
    }
    return line


def bench_cfg5(args, world, rank, local, workload="cfg5"):
    import torch

    from paper_1502_03162_b200 import dist as tdist, synth

    cfg = synth.CONFIGS[workload]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    T = cfg.ny
    # this rank's sources: the direction partition (dist.MixShard); each row is
    # drawn from its global index's own stream, so every N renders the same mix
    shard = tdist.MixShard(ms, sd, T, world=world, rank=rank)
    cnt = int(shard.sources.size)
    y = synth.device_sources_indexed(shard.sources, T, seed=1000) if cnt else \
        torch.empty((0, T), device="cuda")
    mix = shard.mix
    z = shard.alloc_z()
    outb = torch.empty((cfg.ears, (mix.out_len + 3) // 4 * 4), device="cuda")
    shard.render(y, z=z, out=outb)  # builds the plan, validates the inputs once (fused finite check)
    flush = _flush_fn()

    kev = []  # CUDA events around the partial of every step (the dominant kernels)

    def step():  # = shard.render(y, z=z, out=outb): partial -> one reduce -> f on rank 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        zz = shard.partial(y, z=z, check_finite=False)
        e1.record()
        kev.append((e0, e1))
        tdist.reduce_partials(zz, dst=0, group=shard.group)
        if shard.rank == 0:
            shard.mix.finish(zz, out=outb)

    with ClockSampler(local) as clk:
        ms_steps, wall = timed(step, args.steps, args.warmup, world, flush)
    tot = _max_over_ranks(sum(ms_steps), world)
    samples = cfg.sources * cfg.ears * T  # src x ear (one direction per source)
    value = samples * args.steps / (tot * 1e-3)
    # dominant kernel: the rank's partial mix (k_mix_mma + fixup pass + k_mix_finish),
    # CUDA events on the launching stream around it inside every timed step
    kern_ms = sum(a.elapsed_time(b) for a, b in kev[-args.steps:]) / args.steps
    kern_ms_max = _max_over_ranks(kern_ms, world)
    ndist = len(np.unique(sd[shard.sources])) if cnt else 0
    zlen = T + cfg.K - 1
    bytes_local = 4.0 * cnt * T  # every source sample read once
    # executed FLOPs of the g-first algorithm: direction sums + 2 ears x nnz taps per direction and z sample
    flops_local = 2.0 * ndist * cfg.ears * cfg.nnz * zlen + 1.0 * cnt * T
    peaks = _peaks()
    sm = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = sm * FP32_LANES_PER_SM * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12
    achieved = bytes_local / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": _traffic(workload), "peak_src": peaks["src"],
            "kernel": ("k_mix_mma (tcgen05.mma split-fp16 over direction sums, 1 KB TMA source slices) "
                       "+ fixup pass + k_mix_finish") if mix.path == "tensor" else "k_mix (TMEM window + FFMA2)",
            "path": mix.path, "kernel_ms": kern_ms, "kernel_ms_max_over_ranks": kern_ms_max,
            "alg_bytes_per_launch": bytes_local, "sources_on_rank0": cnt, "distinct_directions_rank0": int(ndist),
            "fp32_equiv_tflops": flops_local / (kern_ms * 1e-3) / 1e12,
            "fp32_equiv_frac": flops_local / (kern_ms * 1e-3) / 1e12 / fp32_peak}
    # e2e: the rank's sources from pinned host memory every step (H2D inside
    # the timed region), the mix through the public API, the stereo result
    # back to the host on rank 0
    e2e = None
    if not args.no_e2e:
        try:
            y_pin = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
            y_pin.copy_(y)
            out_pin = torch.empty(outb.shape, dtype=torch.float32, pin_memory=True)

            def e2e_step():
                y.copy_(y_pin, non_blocking=True)
                r = shard.render(y, z=z, out=outb)  # the user's call: includes the fused non-finite check
                if rank == 0:
                    out_pin.copy_(outb, non_blocking=True)
                return r

            ms_e2e, _ = timed(e2e_step, 2, 1, world)
            e2e_ms = _max_over_ranks(sum(ms_e2e), world)
            h2d = float(cfg.sources) * T * 4  # every rank copies its own sources: the whole job's inputs
            e2e = {"value": samples * 2 / (e2e_ms * 1e-3), "unit": "samples/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(out_pin.numel() * 4),
                   "ms_per_step": e2e_ms / 2, "note": "H2D of all sources (PCIe-bound) every step"}
            del y_pin, out_pin
        except RuntimeError as err:  # pinning 47 GB / world of host memory can fail on small hosts
            e2e = {"value": None, "unavailable": "pinned host buffer: %s" % str(err).splitlines()[0]}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Philox source per global index on device; BASELINE laws)",
        "config": workload_config(workload, world),
        "roofline": roof, "e2e": e2e, "gpu_launches": args.steps * (mix.kernels + (1 if rank == 0 else 0)),
        "clocks": clk.summary(),
    }
    return line


def _pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))]


def bench_cfg4(args, world, rank, local, workload="cfg4"):
    """Streaming: 512 sources x 60 s in 256-sample blocks with carried history.
    A step is the whole 60 s stream (11,250 blocks) replayed as one CUDA graph;
    per-block device latency is measured with events around single blocks."""
    import torch

    from paper_1502_03162_b200 import batch, synth

    cfg = synth.CONFIGS[workload]
    B = cfg.block
    T = cfg.ny // B * B
    nblk = T // B
    ms = synth.models(cfg, seed=4)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
    y = synth.device_sources_indexed(np.arange(cfg.sources), T, seed=44 + 1000 * rank)
    st = batch.StreamRenderer(ms, sd, B)
    out = torch.empty((cfg.ears, T), device="cuda")
    # per-block device latency (a GPU sleep ahead of each block hides the host enqueue)
    lat = []
    st.reset()
    for b in range(min(2000, nblk)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        e0.record()
        st.step(y[:, b * B:(b + 1) * B], out=out[:, b * B:(b + 1) * B])
        e1.record()
        e1.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    st.reset()
    g = st.capture(y, out, nblk)
    flush = _flush_fn()

    def step():
        st.reset()
        g.replay()

    with ClockSampler(local) as clk:
        ms_steps, wall = timed(step, args.steps, args.warmup, world, flush)
    tot = _max_over_ranks(sum(ms_steps), world)
    samples = cfg.sources * cfg.ears * T * world
    value = samples * args.steps / (tot * 1e-3)
    # parity of the streamed output against the offline mixdown of the same input
    off = batch.MixRenderer(ms, sd, T).render(y)
    err = float(((out - off[:, :T]).double().norm() / off[:, :T].double().norm()).item())
    per_block_ms = statistics.mean(ms_steps) / nblk
    peaks = _peaks()
    bytes_block = 4.0 * cfg.sources * B
    achieved = bytes_block / (per_block_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": _traffic(workload), "peak_src": peaks["src"],
            "kernel": "k_stream_cl (one launch per block, clusters of 8 CTAs)", "kernel_ms": per_block_ms,
            "alg_bytes_per_launch": bytes_block,
            "note": "latency-bound: 512 KB of new samples per block; the launch, the cluster exchange and "
                    "the cross-cluster ticket set the block time, not HBM"}
    # e2e per block through the public API: pinned host block -> device, step, result -> host
    hin = torch.empty((cfg.sources, B), dtype=torch.float32).pin_memory()
    hout = torch.empty((cfg.ears, B), dtype=torch.float32).pin_memory()
    dblk = torch.empty((cfg.sources, B), device="cuda")
    dout = torch.empty((cfg.ears, B), device="cuda")
    hin.copy_(y[:, :B])
    e2e_lat = []
    st.reset()
    for _ in range(500):
        t0 = time.perf_counter()
        dblk.copy_(hin, non_blocking=True)
        st.step(dblk, out=dout)
        hout.copy_(dout, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        e2e_lat.append(time.perf_counter() - t0)
    e2e_block_s = statistics.median(e2e_lat)
    # the same per block as one CUDA graph (copy in, step, copy out): one host launch per block
    g_io = st.host_step_graph(hin, hout)
    st.reset()
    e2e_glat = []
    for _ in range(500):
        t0 = time.perf_counter()
        g_io.replay()
        torch.cuda.current_stream().synchronize()
        e2e_glat.append(time.perf_counter() - t0)
    e2e_graph_s = statistics.median(e2e_glat)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Philox sources on device; BASELINE laws)",
        "config": workload_config(workload, world),
        "block_latency_us": {"median": statistics.median(lat), "p99": _pct(lat, 0.99), "max": max(lat),
                             "realtime_budget": 1e6 * B / synth.FS_48K},
        "stream": {"blocks": nblk, "us_per_block": 1e3 * per_block_ms, "mode": "CUDA graph of all blocks"},
        "stream_vs_offline_rel_l2": err,
        "roofline": roof,
        "e2e": {"value": cfg.sources * cfg.ears * B / e2e_graph_s, "unit": "samples/s",
                "h2d_bytes_per_step": int(hin.numel() * 4), "d2h_bytes_per_step": int(hout.numel() * 4),
                "step": "one block from pinned host memory and back (median of 500 host round trips): "
                        "StreamRenderer.host_step_graph replayed per block",
                "latency_us": {"median": 1e6 * e2e_graph_s, "p99": 1e6 * _pct(e2e_glat, 0.99)},
                "eager_latency_us": {"median": 1e6 * e2e_block_s, "p99": 1e6 * _pct(e2e_lat, 0.99),
                                     "step": "copy in, StreamRenderer.step, copy out, synchronize"}},
        "gpu_launches": args.steps * nblk, "clocks": clk.summary(),
    }
    return line


def bench_cfg3(args, world, rank, local):
    """Sparsity / length sweep: every point of BASELINE config 3, one render each step."""
    import torch

    from paper_1502_03162_b200 import batch, synth

    peaks = _peaks()
    flush = _flush_fn()
    pts, tot_samples, tot_ms, tot_bytes = [], 0, 0.0, 0.0
    launches = 0
    with ClockSampler(local) as clk:
        for cfg in synth.cfg3_points():
            ms = synth.models(cfg, seed=cfg.K * 1000 + cfg.nnz)
            y = torch.from_numpy(synth.source(cfg.ny, seed=3 + rank).astype(np.float32)).cuda()
            br = batch.BatchRenderer(ms)
            out = br.alloc(cfg.ny)
            br.render_all(y, out=out)
            step_ms, _ = timed(lambda: br.render_all(y, out=out, check_finite=False), args.steps, args.warmup,
                               world, flush)
            t = _max_over_ranks(sum(step_ms), world) / args.steps
            L = br.out_len(cfg.ny)
            samples = cfg.ears * cfg.dirs * L
            bytes_ = 4.0 * samples + 4 * cfg.ny
            pts.append({"point": cfg.name, "K": cfg.K, "nnz": cfg.nnz, "path": br.native.path(), "ms": t,
                        "samples_per_s": samples * world / (t * 1e-3),
                        "hbm_frac": bytes_ / (t * 1e-3) / (peaks["hbm_gbs"] * 1e9)})
            tot_samples += samples * world * args.steps
            tot_ms += t * args.steps
            tot_bytes += bytes_ * args.steps
            launches += args.steps * br.native.kernels(cfg.ny)
            del out, br
    achieved = tot_bytes / (tot_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": tot_samples / (tot_ms * 1e-3), "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; BASELINE laws)", "config": workload_config("cfg3", world),
        "points": pts,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_src": peaks["src"],
                     "kernel": "k_render_mma / k_render per point (aggregate over the sweep)"},
        "e2e": None, "gpu_launches": launches, "clocks": clk.summary(),
    }
    return line


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(n):
    """Re-execute this command under torch.distributed.run with n processes (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr=127.0.0.1", "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + sys.argv[1:]
    os.environ["TOEP_BENCH_SPAWNED"] = "1"
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def _nccl_init_lines(path):
    try:
        with open(path) as fh:
            return [ln.strip() for ln in fh if "Init" in ln or "nRanks" in ln or "comm" in ln][:8]
    except OSError:
        return []


def dry_run(args, world, rank):
    """The multi-rank launch path without a GPU: self-spawn under torchrun,
    one process per "GPU", gloo rendezvous, each rank's share of the cfg5
    sources by direction (dist.MixShard's partition), gathered on rank 0."""
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _spawn(args.gpus)
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    from paper_1502_03162_b200 import dist as tdist, synth
    cfg = synth.CONFIGS["cfg5"]
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    mine = tdist.partition_by_direction(sd, world)[rank]
    share = {"rank": rank, "sources": int(mine.size), "directions": int(np.unique(sd[mine]).size),
             "first": int(mine[0]) if mine.size else -1}
    shares = [share]
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        shares = [None] * world
        dist.all_gather_object(shares, share)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": workload_config("cfg5", world),
                          "shares": shares}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the cfg2 fused_render object at N=1")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU: launch the ranks (gloo), partition the cfg5 sources, print the plan")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist()
    if args.dry_run:
        return dry_run(args, world, rank)

    if args.impl == "reference":
        return run_reference(args, world, rank)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _spawn(args.gpus)  # does not return
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d (launch one process per GPU)" % (args.gpus, world))

    import torch
    torch.cuda.set_device(local)
    nccl = None
    if world > 1:
        import tempfile

        import torch.distributed as dist
        log = os.path.join(tempfile.gettempdir(), "toep_nccl.%d.%d.log" % (os.getpid(), rank))
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", log)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        torch.cuda.synchronize()
        lines = _nccl_init_lines(log)
        for ln in lines:
            sys.stderr.write("[rank %d] %s\n" % (rank, ln))
        nccl = {"backend": dist.get_backend(), "world": dist.get_world_size(),
                "version": ".".join(str(v) for v in torch.cuda.nccl.version()), "init_lines_rank0": lines}
    if args.workload in ("cfg1", "cfg2"):
        line = bench_render(args, world, rank, local, args.workload)
    elif args.workload == "cfg5":
        line = bench_cfg5(args, world, rank, local)
    elif args.workload == "cfg4":
        line = bench_cfg4(args, world, rank, local)
    else:
        line = bench_cfg3(args, world, rank, local)
    if nccl:
        line["nccl"] = nccl
    if world == 1 and args.workload == "cfg5" and not args.no_fused:
        fr = bench_render(args, world, rank, local, "cfg2", steps=min(args.steps, 20), e2e=False)
        line["fused_render"] = {k: fr[k] for k in ("value", "unit", "ms_per_step", "steps", "config", "roofline",
                                                    "gpu_launches", "clocks")}
        line["gpu_launches"] += fr["gpu_launches"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(args.workload)
        for pt in line.get("points", ()):  # cfg3: the reference beside every point
            cpu = line["cpu_baseline"].get("points", {}).get(pt["point"])
            if cpu:
                pt["cpu_samples_per_s"] = cpu
                pt["vs_cpu"] = pt["samples_per_s"] / cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
