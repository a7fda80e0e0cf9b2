"""Measure the B200 cost table behind engine.measured_cost_per_sample / measured_crossover.

    python tools/measure_costs.py [--out paper_1502_03162_b200/data/b200_costs.json]

For |y| = 2,205 (50 ms at 44.1 kHz) and 44,100 (1 s) -- the two signal lengths
of the paper's crossover (engine/__init__.py:278-313) -- and
dense random filters of each size (taps U(0.5, 1.5), y ~ N(0,1): the reference
bench's inputs, engine/__init__.py:327-376):
  * percall: engine.convolve on device-resident tensors, per mode
    (sparse_direct, dense_direct, fft_overlap_save);
  * batched: BatchRenderer.render_all of one signal through 256 directions of
    the same filter size (Lf = 1, so the GEMM-form reflection stage is what
    is timed), per output sample.
Device time only: a GPU sleep is queued ahead of a burst of 20 calls so the
host has enqueued them all before the first starts; CUDA events bracket the
burst (median of the bursts).  Values are ns per output sample.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = {2205: [1, 2, 4, 8, 16, 32, 50, 64, 90, 100, 128, 150, 200, 256, 400, 512, 1024, 2048],
         44100: [1, 2, 4, 8, 16, 32, 64, 100, 124, 128, 150, 200, 256, 400, 512, 1024, 2048, 4096]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_1502_03162_b200", "data", "b200_costs.json"))
    ap.add_argument("--repeats", type=int, default=7)
    args = ap.parse_args()
    import torch

    from paper_1502_03162_b200 import FactorizedModel, SparseFilter, batch, engine

    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    table = {"units": "ns per output sample", "device": torch.cuda.get_device_name(0), "percall": {},
             "batched": {}, "sizes": {}}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def burst(call, samples, calls=20):
        ts = []
        for _ in range(args.repeats):
            torch.cuda.synchronize()
            torch.cuda._sleep(5_000_000)  # ~2.5 ms of GPU time: the host enqueues the burst meanwhile
            ev[0].record()
            for _ in range(calls):
                call()
            ev[1].record()
            ev[1].synchronize()
            ts.append(ev[0].elapsed_time(ev[1]) * 1e6 / (calls * samples))
        return statistics.median(ts)
    for n, sizes in SIZES.items():
        y = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda()
        table["sizes"][str(n)] = sizes
        pc = {m: [] for m in engine.MODES}
        bt = []
        for k in sizes:
            taps = rng.uniform(0.5, 1.5, size=k)
            out_len = n + k - 1
            for mode in engine.MODES:
                plan = engine.ConvPlan(taps, mode)
                engine.convolve(plan, y)
                pc[mode].append(burst(lambda: engine._convolve_device(plan, y), out_len))  # no host-side checks (they sync)
            D = 256
            refl = [SparseFilter(np.arange(k, dtype=np.int64), taps, k) for _ in range(D)]
            br = batch.BatchRenderer([FactorizedModel(np.array([1.0]), refl)])
            out = br.alloc(n)
            br.render_all(y, out=out)
            bt.append(burst(lambda: br.render_all(y, out=out, check_finite=False), D * out_len))
            print(n, k, {m: round(pc[m][-1], 4) for m in pc}, "batched", round(bt[-1], 5), flush=True)
        table["percall"][str(n)] = pc
        table["batched"][str(n)] = bt
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(table, fh, indent=1)
    print(args.out)


if __name__ == "__main__":
    main()
