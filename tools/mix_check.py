"""Quick tensor-core mixdown check: parity vs the oracle on windows, and timing at cfg5 size.

    python tools/mix_check.py [--full]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1502_03162_b200 import batch, synth  # noqa: E402
from paper_1502_03162_b200.batch import model_rows  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check(S, T, nnz=24, dirs=1250, seed=5, scale=1.0, windows=None):
    cfg = synth.Config("c", ny=T, M=200, K=100, nnz=nnz, dirs=dirs, ears=2, sources=S)
    ms = synth.models(cfg, seed=seed)
    sd = synth.source_directions(S, dirs, seed=seed)
    y = synth.device_sources(S, T, seed=seed + 1)
    if scale != 1.0:
        y.mul_(scale)
    mix = batch.MixRenderer(ms, sd, T)
    z = mix.partial(y)
    out = mix.finish(z)
    torch.cuda.synchronize()
    f = np.stack([m.resonance_taps for m in ms])
    rows = model_rows(ms)
    if windows is None:
        windows = [(0, min(T + 199, 3000)), (max(0, T // 2 - 700), 1500), (max(0, T + 199 - 1300), 1300)]
    errs = []
    for t0, W in windows:
        W = min(W, T + 199 - t0)
        lo = max(0, t0 - 199)
        hi = min(T, t0 + W)
        yc = y[:, lo:hi].double().cpu().numpy()
        ref = oracle.mix_window(yc, sd, f, rows, cfg.K, dirs, t0 - lo, W)
        got = out[:, t0:t0 + W].double().cpu().numpy()
        errs.append(max(rel(got[e], ref[e]) for e in range(2)))
    return mix.path, errs


if __name__ == "__main__":
    torch.cuda.set_device(0)
    if "--prof" in sys.argv:  # one cfg5 partial with a TOEP_MIX_PROF build (TOEP_LIB=...); --share R/N: rank R of N
        from paper_1502_03162_b200 import dist as tdist
        cfg = synth.CONFIGS["cfg5"]
        ms = synth.models(cfg, seed=5)
        sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
        if "--share" in sys.argv:
            r, n = (int(v) for v in sys.argv[sys.argv.index("--share") + 1].split("/"))
            mine = tdist.partition_by_direction(sd, n)[r]
            sd = sd[mine]
        y = synth.device_sources(sd.size, cfg.ny, seed=1000)
        mix = batch.MixRenderer(ms, sd, cfg.ny)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        z = mix.alloc_z()
        mix.partial(y, z=z)
        torch.cuda.synchronize()
        print("---- second call", flush=True)
        ev[0].record()
        mix.partial(y, z=z)
        ev[1].record()
        torch.cuda.synchronize()
        print("partial ms %.3f (%d sources)" % (ev[0].elapsed_time(ev[1]), sd.size), flush=True)
        sys.exit(0)
    for S, T, sc in [(6, 3000, 1.0), (192, 100_000, 1.0), (300, 20_000, 1e-9), (300, 20_000, 1e9), (64, 1000, 1.0)]:
        p, e = check(S, T, scale=sc)
        print("S=%d T=%d scale=%g path=%s max rel L2 per window: %s" % (S, T, sc, p, ["%.2e" % x for x in e]), flush=True)
    if "--full" in sys.argv:
        cfg = synth.CONFIGS["cfg5"]
        ms = synth.models(cfg, seed=5)
        sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
        y = synth.device_sources(cfg.sources, cfg.ny, seed=1000)
        for env in ("1", "0"):
            os.environ["TOEP_MIX_MMA"] = env
            mix = batch.MixRenderer(ms, sd, cfg.ny)
            z = mix.alloc_z()
            mix.partial(y, z=z)
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ts = []
            for _ in range(5):
                ev[0].record()
                mix.partial(y, z=z, check_finite=False)
                ev[1].record()
                torch.cuda.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
            print("cfg5 path=%s partial ms: %s  -> %.1f GB/s" % (mix.path, ["%.3f" % t for t in ts],
                                                                 47.19e9 / (min(ts) * 1e-3) / 1e9), flush=True)
            zz = z[:, :mix.z_len]
            bad = (~torch.isfinite(zz)).nonzero()
            print("path=%s non-finite z samples: %d first: %s" % (mix.path, bad.shape[0], bad[:5].tolist()), flush=True)
            if env == "1":
                zt = zz.clone()
                f = np.stack([m.resonance_taps for m in ms])
                rows = model_rows(ms)
                out = mix.finish(z)
                for t0 in (0, 2048 * 700 + 17, cfg.ny - 1000):
                    W = min(1500, cfg.ny + 199 - t0)
                    lo = max(0, t0 - 199)
                    yc = y[:, lo:min(cfg.ny, t0 + W)].double().cpu().numpy()
                    ref = oracle.mix_window(yc, sd, f, rows, cfg.K, cfg.dirs, t0 - lo, W)
                    got = out[:, t0:t0 + W].double().cpu().numpy()
                    print("cfg5 window t0=%d rel L2 %.2e %.2e" % (t0, rel(got[0], ref[0]), rel(got[1], ref[1])), flush=True)
            else:
                a, b = zt.double().cpu().numpy(), zz.double().cpu().numpy()
                print("tensor vs window z rel L2: %.2e" % rel(a, b))
