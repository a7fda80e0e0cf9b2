"""GPU: both stage-2 kernels of toep_renderer_render against the oracle --
the tensor-core GEMM (split-fp16 tcgen05.mma, the default) and the TMEM
window + FFMA2 kernel (selected for very sparse long filters, or forced with
TOEP_RENDER_MMA=0) -- over the cfg3 shape grid at reduced direction count."""
import numpy as np
import pytest

import oracle
from conftest import TOL, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(cuda):
    from paper_1502_03162_b200 import batch, synth
    from paper_1502_03162_b200.batch import model_rows
    return batch, synth, model_rows


def _render_check(mods, cfg, seed, expect_path, ny=30_000, rows=(0, 1, 63, 64, 129, 200, 263)):
    batch, synth, model_rows = mods
    ms = synth.models(cfg, seed=seed)
    y = synth.source(ny, seed=seed + 1)
    br = batch.BatchRenderer(ms)
    assert br.native.path() == expect_path
    out = br.render_all(y)
    f = np.stack([m.resonance_taps for m in ms])
    rows = [r for r in rows if r < cfg.ears * cfg.dirs]
    ref = oracle.render_rows(y, f, model_rows(ms), cfg.K, cfg.dirs, rows=np.asarray(rows, np.int32))
    got = out.reshape(-1, out.shape[-1])[list(rows)].cpu().numpy()
    for i in range(len(rows)):
        assert rel_l2(got[i], ref[i]) <= TOL, (rows[i], rel_l2(got[i], ref[i]))


@pytest.mark.parametrize("K,nnz", [(50, 16), (50, 50), (100, 4), (100, 16), (100, 64), (150, 16), (150, 150)])
def test_tensor_path(mods, K, nnz):
    from paper_1502_03162_b200.synth import Config
    cfg = Config("t", ny=30_000, M=200, K=K, nnz=nnz, dirs=133, ears=2)  # 133: a partial last 128-direction chunk
    _render_check(mods, cfg, K + nnz, "tensor")


@pytest.mark.parametrize("K,nnz", [(100, 16), (150, 8), (150, 4)])
def test_window_path(mods, K, nnz, monkeypatch):
    from paper_1502_03162_b200.synth import Config
    cfg = Config("w", ny=30_000, M=200, K=K, nnz=nnz, dirs=133, ears=2)
    if nnz > 8:
        monkeypatch.setenv("TOEP_RENDER_MMA", "0")  # forced; nnz <= 8 with K > 128 selects it by itself
    _render_check(mods, cfg, 7 * K + nnz, "window")


def test_tensor_path_tiny_and_edges(mods):
    """Signals shorter than one 128-sample tile, and tile-boundary lengths, on the tensor path."""
    batch, synth, model_rows = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("e", ny=100, M=200, K=100, nnz=16, dirs=5, ears=1)
    ms = synth.models(cfg, seed=3)
    br = batch.BatchRenderer(ms)
    assert br.native.path() == "tensor"
    f = np.stack([m.resonance_taps for m in ms])
    for ny in (1, 2, 57, 127, 128, 129, 511, 512, 513):
        y = synth.source(ny, seed=ny)
        out = br.render_all(y).reshape(-1, ny + 199).cpu().numpy()
        ref = oracle.render_rows(y, f, model_rows(ms), cfg.K, cfg.dirs)
        for r in range(cfg.dirs):
            assert rel_l2(out[r], ref[r]) <= TOL, (ny, r)


def test_tensor_path_small_and_large_magnitudes(mods):
    """Power-of-two operand scaling keeps the split exact across magnitudes."""
    batch, synth, model_rows = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=5_000, M=200, K=100, nnz=16, dirs=20, ears=2)
    ms = synth.models(cfg, seed=11)
    br = batch.BatchRenderer(ms)
    f = np.stack([m.resonance_taps for m in ms])
    for scale in (1e-30, 1e-6, 1.0, 1e6, 1e30):
        y = synth.source(cfg.ny, seed=4) * scale
        out = br.render_all(y).reshape(2 * cfg.dirs, -1).cpu().numpy()
        ref = oracle.render_rows(y, f, model_rows(ms), cfg.K, cfg.dirs, rows=np.array([0, 21, 39], np.int32))
        for i, r in enumerate((0, 21, 39)):
            assert rel_l2(out[r], ref[i]) <= TOL, (scale, r)


@pytest.mark.parametrize("K,lf,dirs,ears", [(1, 1, 1, 1), (2, 3, 3, 2), (16, 1, 2, 1), (17, 40, 5, 2), (33, 7, 130, 1),
                                            (128, 73, 4, 2), (129, 20, 3, 2), (192, 9, 2, 1), (200, 1, 2, 2),
                                            (256, 5, 3, 1), (257, 5, 2, 1), (498, 3, 2, 1), (40, 5, 7, 3)])
def test_shape_envelope(mods, K, lf, dirs, ears):
    """Reflection lengths across every kernel boundary (KPAD 16..256, the
    window kernel's KWIN tiers, the banded fallback), tiny resonance filters,
    one ear, a single direction and partial 128-direction chunks."""
    batch, synth, model_rows = mods
    from paper_1502_03162_b200 import FactorizedModel, SparseFilter
    rng = np.random.default_rng(K * 31 + lf)
    models = []
    for e in range(ears):
        refl = []
        for d in range(dirs):
            n = int(rng.integers(1, min(K, 24) + 1))
            idx = np.sort(rng.choice(K, size=n, replace=False)).astype(np.int64)
            refl.append(SparseFilter(idx, np.abs(rng.standard_normal(n)) + 0.05, K))
        models.append(FactorizedModel(rng.standard_normal(lf), refl))
    br = batch.BatchRenderer(models)
    f = np.stack([m.resonance_taps for m in models])
    for ny in (1, 300, 4097):
        y = synth.source(ny, seed=ny + K)
        out = br.render_all(y).reshape(ears * dirs, -1).cpu().numpy()
        ref = oracle.render_rows(y, f, model_rows(models), K, dirs)
        for r in range(ears * dirs):
            assert rel_l2(out[r], ref[r]) <= TOL, (ny, r, br.native.path())


def test_kernel_count_query(mods):
    """toep_renderer_kernels: what bench.py reports as gpu_launches."""
    batch, synth, model_rows = mods
    from paper_1502_03162_b200.synth import Config
    br = batch.BatchRenderer(synth.models(Config("k", ny=1000, M=200, K=100, nnz=16, dirs=8, ears=2), seed=1))
    assert br.native.path() == "tensor"
    assert br.native.kernels(1000) == 1           # small renders: the clustered launch alone
    assert br.native.kernels(441_000) in (1, 2)   # + the fill launch when clusters leave SMs idle
    bw = batch.BatchRenderer(synth.models(Config("w", ny=1000, M=250, K=150, nnz=4, dirs=8, ears=2), seed=1))
    assert bw.native.path() == "window" and bw.native.kernels(441_000) == 1
