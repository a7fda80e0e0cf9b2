"""Seeded synthetic inputs with the shapes and value laws of BASELINE.json's configs.

No dataset is involved (BASELINE names none); SURVEY.md §8(d) fixes the laws:
  * resonance f[n] = N(0,1) * exp(-n/10), n < Lf, L2-normalised (one per ear);
  * reflection g: nnz distinct positions uniform in [0, K), sorted, values
    half-normal |N(0,1)| (redrawn if exactly 0, SparseFilter needs > 0);
  * sources y ~ N(0,1) in fp32.
Host draws use numpy ``default_rng(seed)`` in fp64 and are rounded to fp32 so
the fp64 oracle sees exactly the values the GPU sees.  Long multi-source
signals (configs 4/5) are drawn on the device with torch's Philox generator.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .types import FactorizedModel, SparseFilter

FS_48K = 48_000
T_60S = 60 * FS_48K  # 2,880,000


@dataclass(frozen=True)
class Config:
    name: str
    ny: int          # samples per source
    M: int           # HRIR length = Lf + K - 1
    K: int           # reflection length
    nnz: int         # non-zeros per reflection (== K for the dense control)
    dirs: int
    ears: int
    sources: int = 1
    block: int = 0   # streaming block size (config 4)

    @property
    def lf(self) -> int:
        return self.M - self.K + 1


CONFIGS = {
    "cfg1": Config("cfg1", ny=44_100, M=200, K=100, nnz=12, dirs=1, ears=1),
    "cfg2": Config("cfg2", ny=441_000, M=200, K=100, nnz=16, dirs=1250, ears=2),
    "cfg4": Config("cfg4", ny=T_60S, M=200, K=100, nnz=16, dirs=1250, ears=2, sources=512, block=256),
    "cfg5": Config("cfg5", ny=T_60S, M=200, K=100, nnz=24, dirs=1250, ears=2, sources=4096),
}


def cfg3_points():
    """Sparsity/length sweep: K in {50,100,150} (Lf = 201-K) x nnz in {4..64} + dense control."""
    pts = []
    for K in (50, 100, 150):
        for nnz in (4, 8, 16, 32, 64, K):
            if nnz > K:
                continue  # K=50, nnz=64 is infeasible (more taps than positions)
            pts.append(Config("cfg3_K%d_nnz%d" % (K, nnz), ny=441_000, M=200, K=K, nnz=nnz, dirs=1250, ears=2))
    return pts


def resonance(rng, lf: int) -> np.ndarray:
    n = np.arange(lf)
    f = rng.standard_normal(lf) * np.exp(-n / 10.0)
    f /= np.linalg.norm(f)
    return f.astype(np.float32).astype(np.float64)


def reflection(rng, K: int, nnz: int) -> SparseFilter:
    pos = np.sort(rng.choice(K, size=nnz, replace=False)).astype(np.int64)
    vals = np.abs(rng.standard_normal(nnz))
    while np.any(vals == 0.0):
        z = vals == 0.0
        vals[z] = np.abs(rng.standard_normal(int(z.sum())))
    vals = vals.astype(np.float32).astype(np.float64)
    return SparseFilter(pos, vals, K)


def models(cfg: Config, seed: int = 0):
    """One FactorizedModel per ear (ear e draws from default_rng(seed + 1000 * (e + 1)))."""
    out = []
    for e in range(cfg.ears):
        rng = np.random.default_rng(seed + 1000 * (e + 1))
        f = resonance(rng, cfg.lf)
        refl = [reflection(rng, cfg.K, cfg.nnz) for _ in range(cfg.dirs)]
        out.append(FactorizedModel(f, refl))
    return out


def source(ny: int, seed: int = 0) -> np.ndarray:
    """One N(0,1) source, fp32 values held in an fp64 array."""
    return np.random.default_rng(seed).standard_normal(ny).astype(np.float32).astype(np.float64)


def source_directions(S: int, dirs: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed + 7).integers(0, dirs, size=S).astype(np.int32)


def device_sources(S: int, T: int, seed: int = 0, device: str = "cuda", out=None):
    """[S, T] N(0,1) fp32 sources drawn on the device (Philox, seeded)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    if out is None:
        out = torch.empty((S, T), device=device, dtype=torch.float32)
    out.normal_(generator=g)
    return out


SOURCE_CHUNK = 256  # rows drawn per generator call by device_sources_indexed


def device_sources_indexed(indices, T: int, seed: int = 0, device: str = "cuda", out=None):
    """Rows of the global source set: row i holds source ``indices[i]``, drawn
    on the device (Philox) as part of its chunk of SOURCE_CHUNK consecutive
    global sources, each chunk from its own seeded stream -- so a sharded run
    renders exactly the sources a one-GPU run renders, whatever the split,
    with one generator call per chunk touched."""
    import torch

    idx = np.asarray(indices, dtype=np.int64)
    if out is None:
        out = torch.empty((idx.size, T), device=device, dtype=torch.float32)
    if idx.size == 0:
        return out
    g = torch.Generator(device=device)
    chunks = np.unique(idx // SOURCE_CHUNK)
    buf = torch.empty((SOURCE_CHUNK, T), device=device, dtype=torch.float32)
    pos = torch.as_tensor(np.arange(idx.size), device=device)
    for c in chunks:
        g.manual_seed(int(seed) * 1_000_003 + int(c))
        buf.normal_(generator=g)
        sel = np.flatnonzero(idx // SOURCE_CHUNK == c)
        out[pos[torch.as_tensor(sel, device=device)]] = buf[torch.as_tensor(idx[sel] - c * SOURCE_CHUNK,
                                                                            device=device)]
    return out
