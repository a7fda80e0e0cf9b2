"""Bisect the tensor-core mixdown against the window kernel on growing shapes (debug tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1502_03162_b200 import batch, synth  # noqa: E402


def run(S, T, nnz=24, seed=5):
    cfg = synth.Config("c", ny=T, M=200, K=100, nnz=nnz, dirs=1250, ears=2, sources=S)
    ms = synth.models(cfg, seed=seed)
    sd = synth.source_directions(S, 1250, seed=seed)
    y = synth.device_sources(S, T, seed=seed + 1)
    os.environ["TOEP_MIX_MMA"] = "1"
    a = batch.MixRenderer(ms, sd, T)
    za = a.partial(y)[:, :a.z_len].double()
    os.environ["TOEP_MIX_MMA"] = "0"
    b = batch.MixRenderer(ms, sd, T)
    zb = b.partial(y)[:, :b.z_len].double()
    err = float((za - zb).norm() / zb.norm())
    nf = (~torch.isfinite(za)).nonzero()
    tiles = sorted(set((nf[:, 1] // 256).tolist()))[:10]
    # per-tile error
    n_t = (T + 255) // 256
    pe = []
    for j in range(n_t):
        sl = slice(256 * j, min(256 * (j + 1), a.z_len))
        d = (za[:, sl] - zb[:, sl]).norm() / max(zb[:, sl].norm(), 1e-30)
        pe.append(float(d))
    badt = [j for j, v in enumerate(pe) if not (v < 1e-4)]
    print("S=%d T=%d rel=%.2e nonfinite=%d nf_tiles=%s bad_tiles(%d)=%s" % (S, T, err, nf.shape[0], tiles,
                                                                           len(badt), badt[:12]), flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for S, T in [(4096, 2000), (4096, 20000), (1024, 200000), (4096, 200000), (256, 2880000), (4096, 1000000)]:
        run(S, T)
