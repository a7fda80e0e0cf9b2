#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2|cfg1|cfg3|cfg4|cfg5]
                    [--impl ours|reference]

Default workload is BASELINE config 2 (configs[1]): one 441,000-sample source
rendered through 1,250 directions x 2 ears (nnz 16, K 100, Lf 101) -> 2,500
channels x 441,199 samples per step.  Metric: output samples/s counted as
src x dir x ear.  For N > 1 (torchrun, one rank per GPU) every rank renders
its own independent source through all 2,500 channels (weak scaling: the
per-GPU work is one config-2 render; no collective, outputs stay on their
GPU).  ``--workload cfg5`` benches the 4,096-source
mixdown with sources split across ranks and one NCCL reduce.

``value``     : device-resident throughput, CUDA events around each step on
                the launching stream, L2 flushed (256 MiB write) between steps,
                max over ranks.
``e2e``       : same metric through the public API with host buffers: pinned
                host -> device input copy, render, device -> host copy of every
                output sample, per step.
``roofline``  : dominant kernel's algorithmic bytes (or FLOPs) / its time vs
                MEASURED_PEAKS.json.
``cpu_baseline`` / ``--impl reference``: the reference's own compiled CPU
                kernels (oracle/_ref, built from pkg/src/toepnmf/engine/_kernels.pyx)
                composed as Renderer.render does, on all host cores.
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


def _workload_config(wl, sample):
    """The config keys our arm reports for this workload, plus the reference sample note."""
    from paper_1502_03162_b200 import synth
    cfg = synth.CONFIGS.get(wl, synth.CONFIGS["cfg2"])
    d = {"workload": wl, "sources": cfg.sources, "directions": cfg.dirs, "ears": cfg.ears, "signal_len": cfg.ny,
         "K": cfg.K, "Lf": cfg.lf, "nnz": cfg.nnz}
    if wl in ("cfg1", "cfg2"):
        d["out_len"] = cfg.ny + cfg.M - 1
    d["sample"] = sample
    return d


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    wl = args.workload if args.workload != "cfg3" else "cfg2"
    step, desc, kind, pool, _ = reference_step_factory(wl, cores)
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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE laws)",
        "config": _workload_config(wl, desc),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind, "sample": desc,
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ our arm ------

METRIC = "output samples/s (src x dir x ear)"


def _flush_fn():
    import torch
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def flush():
        buf.fill_(0.0)
    return flush


def bench_cfg2(args, world, rank, local, workload="cfg2"):
    import torch

    from paper_1502_03162_b200 import batch, synth

    cfg = synth.CONFIGS[workload]
    ms_full = synth.models(cfg, seed=2)
    # N GPUs: weak scaling over independent sources -- rank r renders its own
    # source (seed 22 + r) through every (ear, direction), the per-GPU work of
    # one GPU (tier rule: partitioned units, no data-path collective)
    ms = ms_full
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
        ms_steps, wall = timed(step, args.steps, args.warmup, world, flush)
    tot_ms = sum(ms_steps)
    tot_ms_max = _max_over_ranks(tot_ms, world)
    value = samples_global * args.steps / (tot_ms_max * 1e-3)
    kern_ms = statistics.mean(ms_steps)

    # roofline: HBM-bound (4.002 B/sample algorithmic: 4 B written + amortised y, taps)
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
            "fp32_tflops": flops / (kern_ms * 1e-3) / 1e12,
            "alg_bytes_per_launch": alg_bytes}

    # e2e: pinned host buffers, H2D input + D2H of every output sample each step
    e2e = None
    if not args.no_e2e:
        y_pin = torch.from_numpy(y_host).pin_memory()
        out_pin = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        e2e_steps = max(2, min(args.steps, 5))

        def e2e_step():
            y.copy_(y_pin, non_blocking=True)
            r = br.render_all(y, out=out)  # the user's call: includes the fused non-finite check
            out_pin.copy_(out, non_blocking=True)
            return r

        ms_e2e, _ = timed(e2e_step, e2e_steps, 1, world)
        e2e_ms = _max_over_ranks(sum(ms_e2e), world)
        e2e = {"value": samples_global * e2e_steps / (e2e_ms * 1e-3), "unit": "samples/s",
               "h2d_bytes_per_step": int(y_pin.numel() * 4), "d2h_bytes_per_step": int(out_pin.numel() * 4),
               "ms_per_step": e2e_ms / e2e_steps}

    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded: y~N(0,1), f decaying Gaussian, g half-normal at uniform positions)",
        "config": {"workload": workload, "sources": 1, "directions": cfg.dirs, "ears": cfg.ears,
                   "signal_len": cfg.ny, "K": cfg.K, "Lf": cfg.lf, "nnz": cfg.nnz, "out_len": L,
                   "samples_per_step": samples_global,
                   "parallelism": "independent sources x %d (one per GPU)" % world,
                   "l2": "flushed between steps (256 MiB write)"},
        "roofline": roof, "e2e": e2e, "gpu_launches": args.steps * br.native.kernels(cfg.ny),
        "clocks": clk.summary(),
    }
    return line


def bench_cfg5(args, world, rank, local, workload="cfg5"):
    import torch

    from paper_1502_03162_b200 import batch, dist as tdist, synth

    cfg = synth.CONFIGS[workload]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    # sources partitioned by direction: every direction's sources on one rank,
    # ~S/N sources and ~D/N directions per rank (dist.partition_by_direction)
    mine = tdist.partition_by_direction(sd, world)[rank]
    cnt = int(mine.size)
    T = cfg.ny
    y = synth.device_sources(cnt, T, seed=1000 + rank)
    mix = batch.MixRenderer(ms, sd[mine], T)
    z = mix.alloc_z()
    outb = torch.empty((cfg.ears, (mix.out_len + 3) // 4 * 4), device="cuda")
    group = None
    flush = _flush_fn()

    def step():
        z.zero_()
        mix.partial(y, z=z)
        tdist.reduce_partials(z, dst=0, group=group)
        if rank == 0:
            mix.finish(z, out=outb)

    with ClockSampler(local) as clk:
        ms_steps, wall = timed(step, args.steps, args.warmup, world, flush)
    tot = _max_over_ranks(sum(ms_steps), world)
    samples = cfg.sources * cfg.ears * T  # src x ear (one direction per source)
    value = samples * args.steps / (tot * 1e-3)
    # dominant kernel: k_mix (+ its partial reduce), timed alone with CUDA events
    # on the launching stream over a few extra launches after the timed region
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        mix.partial(y, z=z, check_finite=False)
    ev[1].record()
    torch.cuda.synchronize()
    kern_ms = ev[0].elapsed_time(ev[1]) / reps
    # algorithmic work: every source sample read once (4 B); sources sharing a
    # direction are summed in the kernel, then 2 ears x nnz taps per distinct
    # direction and z sample (executed FLOPs of the g-first algorithm)
    ndist = len(np.unique(sd[mine]))
    zlen = T + cfg.K - 1
    flops_local = 2.0 * ndist * cfg.ears * cfg.nnz * zlen + 1.0 * cnt * T
    bytes_local = 4.0 * cnt * T
    peaks = _peaks()
    sm = torch.cuda.get_device_properties(local).multi_processor_count
    fp32_peak = sm * FP32_LANES_PER_SM * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12
    achieved = bytes_local / (kern_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": _traffic(workload),
            "peak_src": "measured", "kernel": "k_mix<112,24> (+k_mix_reduce)", "kernel_ms": kern_ms,
            "alg_bytes_per_launch": bytes_local, "distinct_directions": int(ndist),
            "fp32_tflops": flops_local / (kern_ms * 1e-3) / 1e12,
            "fp32_frac": flops_local / (kern_ms * 1e-3) / 1e12 / fp32_peak}
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
                r = mix.partial(y, z=z)  # the user's call: includes the fused non-finite check
                tdist.reduce_partials(z, dst=0, group=group)
                if rank == 0:
                    mix.finish(z, out=outb)
                    out_pin.copy_(outb, non_blocking=True)
                return r

            ms_e2e, _ = timed(e2e_step, 2, 1, world)
            e2e_ms = _max_over_ranks(sum(ms_e2e), world)
            e2e = {"value": samples * 2 / (e2e_ms * 1e-3), "unit": "samples/s",
                   "h2d_bytes_per_step": int(y_pin.numel() * 4) * world,
                   "d2h_bytes_per_step": int(out_pin.numel() * 4), "ms_per_step": e2e_ms / 2}
            del y_pin, out_pin
        except RuntimeError as err:  # pinning 47 GB / world of host memory can fail on small hosts
            e2e = {"value": None, "unavailable": "pinned host buffer: %s" % str(err).splitlines()[0]}
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Philox sources on device; BASELINE laws)",
        "config": {"workload": workload, "sources": cfg.sources, "signal_len": T, "K": cfg.K, "Lf": cfg.lf,
                   "nnz": cfg.nnz, "ears": cfg.ears,
                   "parallelism": "sources by direction/%d + nccl reduce" % world,
                   "l2": "inputs (47 GB) larger than L2; flushed between steps"},
        "roofline": roof, "e2e": e2e, "gpu_launches": args.steps * (3 if rank == 0 else 2),
        "clocks": clk.summary(),
    }
    return line


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_line(workload):
    cores = os.cpu_count() or 1
    step, desc, kind, pool, single = reference_step_factory(workload if workload in ("cfg1", "cfg2", "cfg4", "cfg5")
                                                            else "cfg2", cores)
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
    return {"value": n / dt, "unit": "samples/s", "cores": cores, "kind": kind,
            "sample": "%s; %d repetitions" % (desc, reps), "seconds": dt,
            "single_core_value": single(3.0), "cpu_model": _cpu_model()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist()

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.workload in ("cfg1", "cfg2"):
        line = bench_cfg2(args, world, rank, local, args.workload)
    elif args.workload == "cfg5":
        line = bench_cfg5(args, world, rank, local)
    else:
        raise SystemExit("workload %s: see tools/sweep_cfg3.py / tools/stream_cfg4.py" % args.workload)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
