"""Config-5 per-rank work measured alone on one GPU (a projection for N GPUs).

    python tools/shard_cfg5.py [--world 8]

Times, for every rank r of an N-GPU run, the mixdown of exactly the sources
`dist.partition_by_direction` gives r (no collective: each share runs alone),
next to the one-GPU time (measured before and after the shares; their mean).
Every measurement follows >= --settle s of back-to-back calls and records the
median SM clock of its timed steps.  The N-GPU step is bounded below by the slowest
share plus the 23 MB NCCL reduce; this measures the share part only.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--settle", type=float, default=1.5, help="seconds of warm-up per share")
    args = ap.parse_args()
    import numpy as np
    import torch

    from bench import ClockSampler, _flush_fn, timed
    from paper_1502_03162_b200 import batch, dist as tdist, synth

    cfg = synth.CONFIGS["cfg5"]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    flush = _flush_fn()
    res = {"world": args.world, "shares": [], "whole": []}

    def measure(mine):
        y = synth.device_sources_indexed(mine, cfg.ny, seed=1000)
        mix = batch.MixRenderer(ms, sd[mine], cfg.ny)
        z = mix.alloc_z()
        # warm-up: >= args.settle seconds of back-to-back calls, so every share
        # (and the whole) is timed in the board's settled power/clock state
        # under its own load, not in the state the previous share left
        step = lambda: mix.partial(y, z=z, check_finite=False)  # noqa: E731
        t_end = time.perf_counter() + args.settle
        while time.perf_counter() < t_end:
            for _ in range(8):
                step()
                flush()
            torch.cuda.synchronize()
        with ClockSampler(0) as clk:
            ms_steps, _ = timed(step, args.steps, 3, 1, flush)
        out = {"sources": int(mine.size), "directions": int(np.unique(sd[mine]).size),
               "ms": statistics.median(ms_steps), "sm_mhz": clk.summary().get("sm_mhz")}
        del y, mix, z
        torch.cuda.empty_cache()
        return out

    # the whole before and after the shares (the board's power state drifts
    # over a run; the projection uses their mean)
    everyone = np.arange(cfg.sources)
    res["whole"].append(measure(everyone))
    for r, mine in enumerate(tdist.partition_by_direction(sd, args.world)):
        res["shares"].append(dict(world=args.world, rank=r, **measure(mine)))
    res["whole"].append(measure(everyone))
    one = statistics.mean(w["ms"] for w in res["whole"])
    worst = max(s["ms"] for s in res["shares"])
    res["one_gpu_ms"] = one
    res["slowest_share_ms"] = worst
    res["share_efficiency"] = one / (args.world * worst)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
