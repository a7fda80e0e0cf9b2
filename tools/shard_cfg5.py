"""Config-5 per-rank work measured alone on one GPU (a projection for N GPUs).

    python tools/shard_cfg5.py [--world 8]

Times, for every rank r of an N-GPU run, the mixdown of exactly the sources
`dist.partition_by_direction` gives r (no collective: each share runs alone),
next to the one-GPU time.  The N-GPU step is bounded below by the slowest
share plus the 23 MB NCCL reduce; this measures the share part only.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    from bench import _flush_fn, timed
    from paper_1502_03162_b200 import batch, dist as tdist, synth

    cfg = synth.CONFIGS["cfg5"]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    flush = _flush_fn()
    res = {"world": args.world, "shares": []}
    for world in (1, args.world):
        parts = tdist.partition_by_direction(sd, world)
        for r, mine in enumerate(parts):
            y = synth.device_sources_indexed(mine, cfg.ny, seed=1000)
            mix = batch.MixRenderer(ms, sd[mine], cfg.ny)
            z = mix.alloc_z()
            # warm-up long enough for the board's power/clock state to settle on this share's load
            ms_steps, _ = timed(lambda: mix.partial(y, z=z, check_finite=False), args.steps, 10, 1, flush)
            res["shares"].append({"world": world, "rank": r, "sources": int(mine.size),
                                  "directions": int(np.unique(sd[mine]).size),
                                  "ms": statistics.median(ms_steps)})
            del y, mix, z
            torch.cuda.empty_cache()
    one = [s["ms"] for s in res["shares"] if s["world"] == 1][0]
    worst = max(s["ms"] for s in res["shares"] if s["world"] == args.world)
    res["one_gpu_ms"] = one
    res["slowest_share_ms"] = worst
    res["share_efficiency"] = one / (args.world * worst)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
