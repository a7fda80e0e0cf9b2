"""GPU: input-independence of the split-fp16 tensor paths (render and mixdown).

The tensor cores see fp16 hi/lo halves of power-of-two-scaled operands; these
tests push the scaling to its edges and compare against the fp64 oracle
(the reference composition, pkg/src/toepnmf/engine/__init__.py:238-260):
  * directions whose gains span 1 .. 1e-9 inside one 128-direction G chunk
    (render: per-direction G exponents for "wide" chunks);
  * signals scaled to 1e-36 and into the fp32 subnormal range (1e-40), and to
    1e30 (render: two-step tile scale; mix: per-tile fixup pass);
  * a loud transient next to near-silence inside one tile;
  * mixdown sources at directions with gains 1e-7 and loud sources compensating.
Bar: relative L2 <= 1e-5 per channel (north_star)."""
import numpy as np
import pytest

import oracle
from conftest import TOL, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(cuda):
    from paper_1502_03162_b200 import FactorizedModel, SparseFilter, batch, synth
    from paper_1502_03162_b200.batch import model_rows
    return batch, synth, model_rows, FactorizedModel, SparseFilter


def _gain_models(mods, dirs, K, nnz, gains, seed):
    batch, synth, model_rows, FactorizedModel, SparseFilter = mods
    rng = np.random.default_rng(seed)
    ms = []
    for e in range(2):
        refl = []
        for d in range(dirs):
            idx = np.sort(rng.choice(K, size=nnz, replace=False)).astype(np.int64)
            vals = (np.abs(rng.standard_normal(nnz)) + 0.05) * gains[d % len(gains)]
            refl.append(SparseFilter(idx, vals.astype(np.float32).astype(np.float64), K))
        ms.append(FactorizedModel(synth.resonance(rng, 101), refl))
    return ms


def _render_rows_check(mods, ms, y, rows):
    batch, synth, model_rows, _, _ = mods
    br = batch.BatchRenderer(ms)
    assert br.native.path() == "tensor"
    out = br.render_all(y)
    K = ms[0].reflection_length
    D = ms[0].num_directions
    f = np.stack([m.resonance_taps for m in ms])
    ref = oracle.render_rows(y, f, model_rows(ms), K, D, rows=np.asarray(rows, np.int32))
    got = out.reshape(2 * D, -1).cpu().numpy()
    for i, r in enumerate(rows):
        err = rel_l2(got[r], ref[i])
        assert err <= TOL, (r, err)


def test_render_direction_gains_span_one_chunk(mods):
    """Gains 1, 1e-3, 1e-6, 1e-7, 1e-9 interleaved in one 128-direction chunk."""
    _, synth, _, _, _ = mods
    gains = [1.0, 1e-3, 1e-6, 1e-7, 1e-9]
    ms = _gain_models(mods, 40, 100, 16, gains, seed=3)
    y = synth.source(20_000, seed=5)
    _render_rows_check(mods, ms, y, rows=list(range(0, 10)) + [40, 43, 44, 79])


@pytest.mark.parametrize("scale", [1e-36, 1e-40, 1e30])
def test_render_extreme_signal_scale(mods, scale):
    """Whole-signal scale down to fp32 subnormals (tile exponent beyond 2^127) and up to 1e30."""
    _, synth, _, _, _ = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("x", ny=6_000, M=200, K=100, nnz=16, dirs=20, ears=2)
    ms = synth.models(cfg, seed=21)
    y = (synth.source(cfg.ny, seed=6) * scale).astype(np.float32).astype(np.float64)
    if scale < 1e-38:
        assert np.any((y != 0) & (np.abs(y) < np.finfo(np.float32).tiny))  # subnormal samples present
    _render_rows_check(mods, ms, y, rows=[0, 7, 19, 20, 39])


def test_render_transient_next_to_silence(mods):
    """A loud burst next to near-silence inside one 128-sample tile."""
    _, synth, _, _, _ = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("t", ny=4_096, M=200, K=100, nnz=16, dirs=12, ears=2)
    ms = synth.models(cfg, seed=31)
    y = synth.source(cfg.ny, seed=7) * 1e-7
    y[1000:1010] = synth.source(10, seed=8) * 1e3
    y = y.astype(np.float32).astype(np.float64)
    _render_rows_check(mods, ms, y, rows=[0, 5, 11, 12, 23])


def _mix_check(mods, ms, sd, y, windows):
    batch, synth, model_rows, _, _ = mods
    mix = batch.MixRenderer(ms, sd, y.shape[1])
    out = mix.render(y)
    assert mix.path == "tensor"
    T = y.shape[1]
    f = np.stack([m.resonance_taps for m in ms])
    yh = y.double().cpu().numpy()
    for t0, W in windows:
        W = min(W, T + 199 - t0)
        ref = oracle.mix_window(yh, sd, f, model_rows(ms), ms[0].reflection_length, ms[0].num_directions, t0, W)
        got = out[:, t0:t0 + W].double().cpu().numpy()
        for e in range(2):
            err = rel_l2(got[e], ref[e])
            assert err <= TOL, (t0, e, err)


@pytest.mark.parametrize("scale", [1e-36, 1e-40, 1e-12, 1e12, 1e30])
def test_mix_extreme_signal_scale(mods, cuda, scale):
    """Every tile outside the launch scale's fp16 window: the fixup pass re-renders it."""
    _, synth, _, _, _ = mods
    torch = cuda
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=6_000, M=200, K=100, nnz=24, dirs=60, ears=2, sources=80)
    ms = synth.models(cfg, seed=41)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=9).double().mul_(scale).float()
    if scale < 1e-38:
        assert bool(((y != 0) & (y.abs() < torch.finfo(torch.float32).tiny)).any())
    _mix_check(mods, ms, sd, y, [(0, 1500), (2_900, 1300), (cfg.ny - 600, 799)])


def test_mix_transient_and_silence(mods, cuda):
    """Quiet tiles (1e-9) around a loud passage: tiles far below the launch
    scale that still matter are re-rendered at their own scale."""
    _, synth, _, _, _ = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=8_192, M=200, K=100, nnz=24, dirs=50, ears=2, sources=70)
    ms = synth.models(cfg, seed=42)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=10)
    y[:, :3000].mul_(1e-9)
    y[:, 5000:].mul_(1e-9)
    _mix_check(mods, ms, sd, y, [(0, 2800), (2_900, 400), (3_100, 1800), (5_050, 3000)])


def test_mix_direction_gains(mods, cuda):
    """Directions with gains down to 1e-7; the sources at the quiet directions 1e7
    louder, so every direction contributes equally to the mix."""
    _, synth, _, _, _ = mods
    gains = [1.0, 1e-4, 1e-7]
    ms = _gain_models(mods, 30, 100, 24, gains, seed=7)
    S, T = 90, 5_000
    sd = (np.arange(S) % 30).astype(np.int32)
    y = synth.device_sources(S, T, seed=12)
    for s in range(S):
        y[s].mul_(1.0 / gains[int(sd[s]) % 3])
    _mix_check(mods, ms, sd, y, [(0, 2000), (3_000, 2199)])


@pytest.mark.parametrize("mma", ["1", "0"])
def test_mix_paths_shapes(mods, cuda, monkeypatch, mma):
    """Both mixdown kernels (tensor, TMEM-window FFMA2) on shapes around their
    limits: one ear, K = 8 / 50 / 100 / 200 (one ear at K = 200 takes the
    13-chunk, 8-window instantiation of k_mix_mma), one source, sources not a
    multiple of 4, a sub-range partial (s0, count) and T below one tile."""
    batch, synth, model_rows, _, _ = mods
    torch = cuda
    monkeypatch.setenv("TOEP_MIX_MMA", mma)
    from paper_1502_03162_b200.synth import Config
    for K, ears, S, T in [(100, 1, 37, 3_001), (8, 2, 5, 700), (50, 2, 1, 2_000), (100, 2, 9, 100),
                          (200, 1, 23, 2_500)]:
        cfg = Config("p", ny=T, M=K + 100, K=K, nnz=min(K, 8), dirs=17, ears=ears, sources=S)
        ms = synth.models(cfg, seed=K + S)
        sd = synth.source_directions(S, cfg.dirs, seed=S)
        Tp = (T + 3) // 4 * 4  # rows 16-byte aligned (the C ABI's contract for the source array)
        y = torch.zeros((S, Tp), device="cuda")
        y[:, :T] = synth.device_sources(S, T, seed=T)
        y = y[:, :T]
        mix = batch.MixRenderer(ms, sd, T)
        assert mix.path == ("tensor" if mma == "1" else "window")
        out = mix.render(y)
        f = np.stack([m.resonance_taps for m in ms])
        ref = oracle.mix_window(y.double().cpu().numpy(), sd, f, model_rows(ms), K, cfg.dirs, 0, T + cfg.M - 1)
        for e in range(ears):
            assert rel_l2(out[e].double().cpu().numpy(), ref[e]) <= TOL, (K, ears, S, T, e)
        if S >= 5:  # sub-range partial: sources [2, S-1)
            z = mix.partial(y[2:S - 1], s0=2, count=S - 3)
            o2 = mix.finish(z)
            ref2 = oracle.mix_window(y[2:S - 1].double().cpu().numpy(), sd[2:S - 1], f, model_rows(ms), K, cfg.dirs,
                                     0, T + cfg.M - 1)
            for e in range(ears):
                assert rel_l2(o2[e].double().cpu().numpy(), ref2[e]) <= TOL, ("sub", K, e)


def test_mix_many_sources_kstep_groups(mods, cuda):
    """6,000 sources over 1,250 directions: more than 96 K-steps per tile, so
    the tensor mix accumulates a tile in groups (the first stores, the others
    add) -- the accumulation error stays bounded whatever the source count."""
    batch, synth, model_rows, _, _ = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("g", ny=3_000, M=200, K=100, nnz=24, dirs=1250, ears=2, sources=6000)
    ms = synth.models(cfg, seed=77)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=8)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=13)
    _mix_check(mods, ms, sd, y, [(0, 1000), (1_400, 900), (cfg.ny - 700, 899)])
