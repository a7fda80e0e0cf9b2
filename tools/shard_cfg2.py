"""Config-2 per-rank work measured alone on one GPU (a projection for N GPUs).

    python tools/shard_cfg2.py [--world 8]

bench.py --gpus N splits the output time range: rank r renders all 2,500
channels for samples [t0, t1) from y[t0 - (M-1), t1).  This times each
share alone (no collective exists on this path) next to the full render.
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
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import numpy as np
    import torch

    from bench import _flush_fn, timed
    from paper_1502_03162_b200 import batch, synth

    cfg = synth.CONFIGS["cfg2"]
    ms = synth.models(cfg, seed=2)
    y_full = synth.source(cfg.ny, seed=22).astype(np.float32)
    br = batch.BatchRenderer(ms)
    flush = _flush_fn()
    M = cfg.lf + cfg.K - 1
    L = cfg.ny + M - 1
    res = {"world": args.world, "shares": []}
    for world in (1, 2, 4, args.world):
        seg = -(-L // world)
        worst = 0.0
        for r in (0, world - 1):
            t0, t1 = min(L, r * seg), min(L, (r + 1) * seg)
            lo = max(0, t0 - (M - 1))
            hi = max(min(cfg.ny, t1), lo + 1)
            y = torch.from_numpy(np.ascontiguousarray(y_full[lo:hi])).cuda()
            out = br.alloc(y.numel())
            ms_steps, _ = timed(lambda: br.render_all(y, out=out, check_finite=False), args.steps, 3, 1, flush)
            worst = max(worst, statistics.mean(ms_steps))
            del out
        res["shares"].append({"world": world, "slowest_share_ms": worst})
    one = res["shares"][0]["slowest_share_ms"]
    for s in res["shares"]:
        s["efficiency"] = one / (s["world"] * s["slowest_share_ms"])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
