"""BASELINE config 3: sparsity / length sweep on one B200.

    python tools/sweep_cfg3.py [--steps 10] [--check] [--only 150:16,100:16]

y = 441,000 samples, 1,250 directions x 2 ears, K in {50, 100, 150}
(Lf = 201 - K), nnz in {4, 8, 16, 32, 64} plus the dense control nnz = K
(K=50, nnz=64 is infeasible and skipped).  Per point: output samples/s
(src x dir x ear), the binding roofline (HBM write vs FP32 FFMA, ridge =
FP32 peak / HBM peak) and its fraction.  One JSON line per point.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", action="store_true", help="oracle parity on 4 rows per point")
    ap.add_argument("--only", default="", help="comma list of K:nnz points, e.g. 150:16,150:150")
    args = ap.parse_args()
    only = {tuple(int(v) for v in p.split(":")) for p in args.only.split(",") if p}
    import torch

    from bench import _peaks, timed, _flush_fn
    from paper_1502_03162_b200 import batch, synth

    peaks = _peaks()
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    fp32 = sm * 128 * 2 * peaks["sm_max_mhz"] * 1e6
    flush = _flush_fn()
    for cfg in synth.cfg3_points():
        if only and (cfg.K, cfg.nnz) not in only:
            continue
        ms = synth.models(cfg, seed=cfg.K * 1000 + cfg.nnz)
        y = torch.from_numpy(synth.source(cfg.ny, seed=3).astype(np.float32)).cuda()
        br = batch.BatchRenderer(ms)
        out = br.alloc(cfg.ny)
        br.render_all(y, out=out)
        step_ms, _ = timed(lambda: br.render_all(y, out=out, check_finite=False), args.steps, args.warmup, 1, flush)
        t = statistics.mean(step_ms) * 1e-3
        L = br.out_len(cfg.ny)
        samples = cfg.ears * cfg.dirs * L
        flops = 2.0 * cfg.nnz * samples + 2.0 * cfg.ears * cfg.lf * (cfg.ny + cfg.M)
        bytes_ = 4.0 * samples + 4 * cfg.ny
        hbm_frac = bytes_ / t / (peaks["hbm_gbs"] * 1e9)
        fma_frac = flops / t / fp32
        path = br.native.path()
        # the tensor-core path executes the dense GEMM far below its tensor peak, so
        # the output write stream binds it; the FFMA paths bind at HBM or FP32
        if path == "tensor":
            bound = "hbm"
        else:
            bound = "hbm" if flops / bytes_ < fp32 / (peaks["hbm_gbs"] * 1e9) else "fp32"
        line = {"point": cfg.name, "K": cfg.K, "nnz": cfg.nnz, "Lf": cfg.lf, "path": path, "ms": t * 1e3,
                "samples_per_s": samples / t, "bound": bound, "hbm_frac": hbm_frac, "fp32_frac": fma_frac,
                "roofline_frac": hbm_frac if bound == "hbm" else fma_frac}
        if args.check:
            import oracle
            from paper_1502_03162_b200.batch import model_rows
            rows = [0, cfg.dirs - 1, cfg.dirs, 2 * cfg.dirs - 1]
            f = np.stack([m.resonance_taps for m in ms])
            ref = oracle.render_rows(synth.source(cfg.ny, seed=3), f, model_rows(ms), cfg.K, cfg.dirs, rows=rows)
            got = out[:, :, :L].reshape(-1, L)[rows].cpu().numpy()
            line["max_rel_l2"] = max(float(np.linalg.norm(got[i] - ref[i]) / np.linalg.norm(ref[i]))
                                     for i in range(len(rows)))
        print(json.dumps(line), flush=True)
        del out, br


if __name__ == "__main__":
    main()
