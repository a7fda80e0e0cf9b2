"""BASELINE config 4: low-latency streaming mixdown.

    python tools/stream_cfg4.py [--seconds 60] [--latency-blocks 2000]

512 sources x 60 s at 48 kHz (device-resident, Philox-seeded), each at a
uniform-random direction of 1,250 (K=100, nnz 16), per-ear f of 101 taps,
256-sample blocks with carried overlap history (11,250 blocks), summed to a
stereo output.  Reports
  * per-block device latency (CUDA events around each launch; median, p99),
  * end-to-end per-block latency with host I/O (pinned host block -> H2D ->
    step -> D2H of the 2 x 256 output), median and p99,
  * sustained samples/s over the whole stream (src x ear),
  * the same mixdown rendered offline in one call, and the streamed output's
    relative L2 error against it.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=60.0)
    ap.add_argument("--latency-blocks", type=int, default=2000)
    args = ap.parse_args()
    import torch

    from paper_1502_03162_b200 import batch, synth

    cfg = synth.CONFIGS["cfg4"]
    B = cfg.block
    T = int(args.seconds * synth.FS_48K) // B * B
    ms = synth.models(cfg, seed=4)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
    y = synth.device_sources(cfg.sources, T, seed=44)
    nblk = T // B
    st = batch.StreamRenderer(ms, sd, B)
    out = torch.empty((cfg.ears, T), device="cuda")
    # per-block device latency: a GPU sleep ahead of each step hides the host
    # enqueue time, so the events bracket only the kernel
    lat = []
    st.reset()
    for b in range(min(args.latency_blocks, nblk)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)
        e0.record()
        st.step(y[:, b * B:(b + 1) * B], out=out[:, b * B:(b + 1) * B])
        e1.record()
        e1.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    # sustained: the whole stream as one CUDA graph (11,250 kernel nodes)
    st.reset()
    g = st.capture(y, out, nblk)
    st.reset()
    g.replay()  # warm
    torch.cuda.synchronize()
    st.reset()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    total_ms = e0.elapsed_time(e1)
    samples = cfg.sources * cfg.ears * T
    # end-to-end with host I/O for a sample of blocks
    hin = torch.empty((cfg.sources, B), dtype=torch.float32).pin_memory()
    hout = torch.empty((cfg.ears, B), dtype=torch.float32).pin_memory()
    dblk = torch.empty((cfg.sources, B), device="cuda")
    dout = torch.empty((cfg.ears, B), device="cuda")
    hin.copy_(y[:, :B])
    e2e = []
    for b in range(500):
        t0 = time.perf_counter()
        dblk.copy_(hin, non_blocking=True)
        st.step(dblk, out=dout)
        hout.copy_(dout, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        e2e.append((time.perf_counter() - t0) * 1e6)
    # offline reference for the same input (one call) and stream parity
    mix = batch.MixRenderer(ms, sd, T)
    torch.cuda.synchronize()
    o0, o1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    o0.record()
    off = mix.render(y)
    o1.record()
    torch.cuda.synchronize()
    err = float(((out - off[:, :T]).double().norm() / off[:, :T].double().norm()).item())
    line = {
        "workload": "cfg4", "sources": cfg.sources, "block": B, "blocks": nblk, "seconds": T / synth.FS_48K,
        "device_latency_us": {"median": statistics.median(lat), "p99": pct(lat, 0.99), "max": max(lat)},
        "e2e_latency_us_host_io": {"median": statistics.median(e2e), "p99": pct(e2e, 0.99)},
        "realtime_budget_us": 1e6 * B / synth.FS_48K,
        "stream_samples_per_s": samples / (total_ms * 1e-3), "stream_ms_total": total_ms,
        "stream_us_per_block": 1e3 * total_ms / nblk, "stream_mode": "CUDA graph of all blocks",
        "stream_wall_s": wall, "offline_ms": o0.elapsed_time(o1),
        "offline_samples_per_s": samples / (o0.elapsed_time(o1) * 1e-3),
        "stream_vs_offline_rel_l2": err, "gpu_launches_per_block": 1,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
