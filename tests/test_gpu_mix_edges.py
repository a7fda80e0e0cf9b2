"""GPU: the one-pass bucketed mixdown (k_mix) at its edges, and the fused
non-finite input check (the reference's DataError for inf/NaN samples,
engine/__init__.py:162-165) on the render, mix and streaming paths."""
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


def _mix_check(mods, cfg, sd, seed, windows):
    batch, synth, model_rows = mods
    ms = synth.models(cfg, seed=seed)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=seed + 1)
    out = batch.MixRenderer(ms, sd, cfg.ny).render(y)
    yh = y.cpu().numpy().astype(np.float64)
    f = np.stack([m.resonance_taps for m in ms])
    for t0, W in windows:
        ref = oracle.mix_window(yh, sd, f, model_rows(ms), cfg.K, cfg.dirs, t0, W)
        got = out[:, t0:t0 + W].cpu().numpy()
        for e in range(cfg.ears):
            assert rel_l2(got[e], ref[e]) < TOL, (t0, e)


def test_large_buckets(mods):
    """Few directions: buckets of ~12 sources (beyond the 3 prefetched slots)."""
    from paper_1502_03162_b200.synth import Config
    cfg = Config("b", ny=20_000, M=200, K=100, nnz=24, dirs=8, ears=2, sources=96)
    sd = np.random.default_rng(3).integers(0, cfg.dirs, size=cfg.sources).astype(np.int32)
    _mix_check(mods, cfg, sd, 101, [(0, 2500), (9_000, 2100), (cfg.ny - 300, 499)])


def test_one_direction_many_sources(mods):
    """One direction with 2,100 sources: split into buckets of <= 1,024 (the shared-memory source table)."""
    from paper_1502_03162_b200.synth import Config
    cfg = Config("o", ny=3_000, M=200, K=100, nnz=16, dirs=4, ears=2, sources=2100)
    sd = np.full(cfg.sources, 2, np.int32)
    _mix_check(mods, cfg, sd, 202, [(0, 3199)])


def test_bucket_groups_shrink_to_fit_table(mods):
    """~75 sources per direction: 16-bucket groups would hold ~1,200 sources, so the host halves the group."""
    from paper_1502_03162_b200.synth import Config
    cfg = Config("g", ny=2_500, M=200, K=100, nnz=24, dirs=40, ears=2, sources=3000)
    sd = np.random.default_rng(4).integers(0, cfg.dirs, size=cfg.sources).astype(np.int32)
    _mix_check(mods, cfg, sd, 303, [(0, 900), (2_000, 699)])


def test_mono_and_uneven_nnz(mods):
    """One ear, ragged tap counts (generic tap loop), K=150 (KWIN 240)."""
    batch, synth, model_rows = mods
    from paper_1502_03162_b200 import FactorizedModel, SparseFilter
    rng = np.random.default_rng(9)
    K, D = 150, 40
    refl = []
    for d in range(D):
        n = int(rng.integers(0, 20))
        idx = np.sort(rng.choice(K, size=n, replace=False)).astype(np.int64)
        refl.append(SparseFilter(idx, np.abs(rng.standard_normal(n)) + 0.1, K))
    m = FactorizedModel(rng.standard_normal(51), refl)
    sd = rng.integers(0, D, size=64).astype(np.int32)
    y = synth.device_sources(64, 9_000, seed=5)
    out = batch.MixRenderer([m], sd, 9_000).render(y)
    ref = oracle.mix_window(y.cpu().numpy().astype(np.float64), sd, m.resonance_taps[None], model_rows([m]), K, D,
                            0, 9_000 + 199)
    assert rel_l2(out[0].cpu().numpy(), ref[0]) < TOL


def test_nonfinite_detected_in_kernels(mods, cuda):
    batch, synth, _ = mods
    torch = cuda
    from paper_1502_03162_b200 import DataError
    from paper_1502_03162_b200.synth import Config
    cfg = Config("n", ny=8_000, M=200, K=100, nnz=16, dirs=10, ears=2, sources=12, block=256)
    ms = synth.models(cfg, seed=3)
    br = batch.BatchRenderer(ms)
    y = torch.randn(cfg.ny, device="cuda")
    br.render_all(y)
    for bad in (float("nan"), float("inf"), -float("inf")):
        yb = y.clone()
        yb[4321] = bad
        with pytest.raises(DataError, match="non-finite"):
            br.render_all(yb)
    br.render_all(y)  # the flag does not leak into the next call
    br.render_all(yb, check_finite=False)
    br.render_all(y)

    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=1)
    mix = batch.MixRenderer(ms, sd, cfg.ny)
    ys = synth.device_sources(cfg.sources, cfg.ny, seed=2)
    mix.render(ys)
    for pos in (0, 2047, 5000, cfg.ny - 1):  # first tile, tile seam, interior, last sample
        ysb = ys.clone()
        ysb[7, pos] = float("nan")
        with pytest.raises(DataError, match="non-finite"):
            mix.render(ysb)
    mix.render(ys)

    st = batch.StreamRenderer(ms, sd, 256)
    st.step(ys[:, :256].contiguous())
    assert not st.nonfinite()
    blk = ys[:, 256:512].clone()
    blk[3, 17] = float("inf")
    st.step(blk)
    assert st.nonfinite()
    assert not st.nonfinite()  # reading clears it


@pytest.mark.parametrize("kernel", ["cluster", "ticketed"])
@pytest.mark.parametrize("K,ears,block,sources", [(150, 1, 128, 40), (50, 2, 64, 40), (100, 2, 4, 40),
                                                  (100, 2, 256, 2000), (100, 2, 36, 7), (100, 2, 256, 1)])
def test_streaming_shapes(mods, cuda, monkeypatch, K, ears, block, sources, kernel):
    """Streaming blocks against the offline mixdown for other filter lengths,
    one ear, small and odd blocks (empty cluster slices), a source count that
    leaves padding CTAs, many clusters (2,000 sources: 125 clusters in the
    cross-cluster level) -- both streaming kernels (k_stream_cl, and
    k_stream_step with TOEP_STREAM_CLUSTER=0)."""
    monkeypatch.setenv("TOEP_STREAM_CLUSTER", "1" if kernel == "cluster" else "0")
    batch, synth, _ = mods
    torch = cuda
    from paper_1502_03162_b200.synth import Config
    cfg = Config("s", ny=block * 37, M=200, K=K, nnz=12, dirs=60, ears=ears, sources=sources, block=block)
    ms = synth.models(cfg, seed=K + block)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=3)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=9)
    offline = batch.MixRenderer(ms, sd, cfg.ny).render(y)
    st = batch.StreamRenderer(ms, sd, block)
    full = torch.empty((ears, cfg.ny), device="cuda")
    for b in range(cfg.ny // block):
        st.step(y[:, b * block:(b + 1) * block], out=full[:, b * block:(b + 1) * block])
    from conftest import rel_l2 as _rel
    assert _rel(full.cpu().numpy(), offline[:, :cfg.ny].cpu().numpy()) < TOL
