"""CUDA path vs the fp64 oracle on BASELINE-shaped seeded inputs.

Bar (BASELINE.json north_star): relative L2 error <= 1e-5 per channel against
the reference's CPU direct convolution.  Full-size configs are checked on a
row subset against the oracle plus a size-independent identity on every row:
the sum of a full linear convolution equals the product of the operands'
sums, so sum_t out[e,d,t] = sum(y) * sum(f_e) * sum(g_ed).
"""
import numpy as np
import pytest

import oracle
from conftest import TOL, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(cuda):
    from paper_1502_03162_b200 import batch, engine, synth
    return batch, engine, synth


def _rows(models):
    from paper_1502_03162_b200.batch import model_rows
    return model_rows(models)


def _check_rows(out, y, models, rows, K, dirs):
    f = np.stack([m.resonance_taps for m in models])
    ref = oracle.render_rows(y, f, _rows(models), K, dirs, rows=np.asarray(rows, np.int32))
    got = out.reshape(-1, out.shape[-1])[np.asarray(rows)].cpu().numpy()
    errs = [rel_l2(got[i], ref[i]) for i in range(len(rows))]
    return max(errs)


def _check_sums(out, y, models):
    """sum(out_row) == sum(y)*sum(f_e)*sum(g_row) for every row; a dropped or
    misplaced tap moves a row sum by ~|sum(y) sum(f) v|, far above the bound."""
    sy = float(np.sum(y))
    got = out.double().sum(dim=-1).cpu().numpy()  # [E, D]
    l1 = out.double().abs().sum(dim=-1).cpu().numpy()
    for e, m in enumerate(models):
        want = sy * float(np.sum(m.resonance_taps)) * np.array([np.sum(r.values) for r in m.reflections])
        assert np.all(np.abs(got[e] - want) <= 1e-6 * l1[e] + 1e-9)


def test_cfg1_single_channel(mods):
    batch, engine, synth = mods
    cfg = synth.CONFIGS["cfg1"]
    ms = synth.models(cfg, seed=1)
    y = synth.source(cfg.ny, seed=11)
    br = batch.BatchRenderer(ms)
    out = br.render_all(y)
    assert out.shape == (1, 1, 44_299)
    assert _check_rows(out, y, ms, [0], cfg.K, cfg.dirs) < TOL
    # the drop-in per-call path gives the same answer
    got = engine.Renderer(ms[0]).render(y, 0)
    ref = oracle.render_rows(y, ms[0].resonance_taps[None], _rows(ms), cfg.K, 1)[0]
    assert got.shape == ref.shape and rel_l2(got, ref) < TOL


def test_cfg2_full_size(mods):
    batch, _, synth = mods
    cfg = synth.CONFIGS["cfg2"]
    ms = synth.models(cfg, seed=2)
    y = synth.source(cfg.ny, seed=22)
    br = batch.BatchRenderer(ms)
    out = br.render_all(y)
    assert out.shape == (2, 1250, 441_199)
    rows = list(range(0, 2500, 97)) + [1249, 1250, 2499]
    assert _check_rows(out, y, ms, rows, cfg.K, cfg.dirs) < TOL
    _check_sums(out, y, ms)
    # counters follow Renderer.counters semantics (engine/__init__.py:262-269)
    assert br.counters["reflection_macs"] == 2500 * 16 * (cfg.ny + cfg.lf - 1)
    assert br.counters["resonance_macs"] == 2 * cfg.lf * cfg.ny


@pytest.mark.parametrize("K,nnz", [(50, 4), (50, 50), (100, 8), (100, 32), (100, 64), (100, 100),
                                   (150, 16), (150, 64), (150, 150)])
def test_cfg3_sweep_points(mods, K, nnz):
    batch, _, synth = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("p", ny=441_000, M=200, K=K, nnz=nnz, dirs=40, ears=2)
    ms = synth.models(cfg, seed=K * 1000 + nnz)
    y = synth.source(cfg.ny, seed=3)
    out = batch.BatchRenderer(ms).render_all(y)
    assert _check_rows(out, y, ms, [0, 7, 39, 40, 41, 79], K, cfg.dirs) < TOL


def test_ragged_and_empty_rows(mods):
    """Variable nnz per row (incl. empty filters, pkg/tests/test_sparsify.py:227-229)."""
    batch, _, synth = mods
    from paper_1502_03162_b200 import FactorizedModel, SparseFilter
    rng = np.random.default_rng(5)
    K, lf, D = 100, 101, 37
    refl = []
    for d in range(D):
        n = [0, 1, 3, 16, 99, 100][d % 6]
        pos = np.sort(rng.choice(K, n, replace=False))
        refl.append(SparseFilter(pos, rng.uniform(0.1, 1.0, n), K))
    ms = [FactorizedModel(synth.resonance(rng, lf), refl), FactorizedModel(synth.resonance(rng, lf), refl[::-1])]
    y = synth.source(5000, seed=9)
    out = batch.BatchRenderer(ms).render_all(y)
    assert _check_rows(out, y, ms, list(range(2 * D)), K, D) < TOL
    assert float(out[0, 0].abs().max()) == 0.0  # empty filter renders silence


@pytest.mark.parametrize("ny", [1, 2, 15, 16, 17, 100, 2047, 2048, 2049, 4097])
def test_short_and_ragged_signals(mods, ny):
    batch, _, synth = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("s", ny=ny, M=200, K=100, nnz=16, dirs=5, ears=2)
    ms = synth.models(cfg, seed=ny)
    y = synth.source(ny, seed=ny + 1)
    out = batch.BatchRenderer(ms).render_all(y)
    assert out.shape[-1] == ny + 199
    assert _check_rows(out, y, ms, list(range(10)), 100, 5) < TOL


def test_long_reflection_generic_path(mods):
    """K > 497 takes the banded kernel (render and plugin conv_sparse)."""
    batch, engine, synth = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("g", ny=20_000, M=1600, K=1500, nnz=40, dirs=6, ears=2)
    ms = synth.models(cfg, seed=4)
    y = synth.source(cfg.ny, seed=5)
    out = batch.BatchRenderer(ms).render_all(y)
    assert _check_rows(out, y, ms, list(range(12)), cfg.K, cfg.dirs) < TOL
    sf = ms[0].reflections[0]
    got = engine.convolve(engine.ConvPlan(sf, "sparse_direct"), y)
    ref, _ = oracle.conv_sparse(y, sf.indices, sf.values, sf.length)
    assert rel_l2(got, ref) < TOL


@pytest.mark.parametrize("ntaps,ny", [(1, 1), (3, 1), (1, 5000), (101, 441), (700, 3000), (2000, 5000)])
def test_plugin_conv_dense(mods, ntaps, ny):
    _, _, _ = mods
    from paper_1502_03162_b200 import _kernels_cuda
    rng = np.random.default_rng(ntaps * 7 + ny)
    y, h = rng.standard_normal(ny), rng.standard_normal(ntaps)
    got, macs = _kernels_cuda.conv_dense(y, h)
    ref, rmacs = oracle.conv_dense(y, h)
    assert macs == rmacs and got.shape == ref.shape and rel_l2(got, ref) < TOL


def test_plugin_conv_sparse_kernels_agree_with_reference(mods):
    from paper_1502_03162_b200 import _kernels_cuda
    rng = np.random.default_rng(3)
    for length in (1, 4, 100, 113, 114, 241, 242, 497, 498, 3000):
        nnz = min(length, 12)
        idx = np.sort(rng.choice(length, nnz, replace=False))
        vals = rng.uniform(0.1, 2.0, nnz)
        y = rng.standard_normal(1000)
        got, macs = _kernels_cuda.conv_sparse(y, idx, vals, length)
        ref, rmacs = oracle.conv_sparse(y, idx, vals, length)
        assert macs == rmacs and got.shape == ref.shape and rel_l2(got, ref) < TOL, length


def test_mix_offline_window_parity(mods, cuda):
    """Reduced config 5: 192 sources x 100k samples, nnz 24, windows vs oracle."""
    batch, _, synth = mods
    torch = cuda
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=100_000, M=200, K=100, nnz=24, dirs=1250, ears=2, sources=192)
    ms = synth.models(cfg, seed=55)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=77)
    mix = batch.MixRenderer(ms, sd, cfg.ny)
    out = mix.render(y)
    assert out.shape == (2, cfg.ny + 199)
    yh = y.cpu().numpy().astype(np.float64)
    f = np.stack([m.resonance_taps for m in ms])
    for t0, W in [(0, 3000), (51_234, 2500), (cfg.ny - 1000, 1199)]:
        ref = oracle.mix_window(yh, sd, f, _rows(ms), cfg.K, cfg.dirs, t0, W)
        got = out[:, t0:t0 + W].cpu().numpy()
        for e in range(2):
            assert rel_l2(got[e], ref[e]) < TOL, (t0, e)
    torch.cuda.synchronize()


def test_mix_partials_add(mods):
    """Linearity: partial mixes over a source split add up to the whole (the multi-GPU contract)."""
    batch, _, synth = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=30_000, M=200, K=100, nnz=16, dirs=100, ears=2, sources=300)
    ms = synth.models(cfg, seed=56)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=6)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=78)
    mix = batch.MixRenderer(ms, sd, cfg.ny)
    whole = mix.partial(y)
    z = mix.alloc_z()
    parts = []
    for s0, n in [(0, 100), (100, 150), (250, 50)]:
        parts.append(mix.partial(y[s0:s0 + n], s0=s0, count=n))
    total = sum(parts)
    assert rel_l2(total[:, :mix.z_len].cpu().numpy(), whole[:, :mix.z_len].cpu().numpy()) < TOL
    del z


def test_streaming_equals_offline(mods, cuda):
    """Config-4 semantics at reduced size: blocks of 256 with carried history."""
    batch, _, synth = mods
    torch = cuda
    from paper_1502_03162_b200.synth import Config
    cfg = Config("st", ny=256 * 40, M=200, K=100, nnz=16, dirs=1250, ears=2, sources=96, block=256)
    ms = synth.models(cfg, seed=57)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=7)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=79)
    offline = batch.MixRenderer(ms, sd, cfg.ny).render(y)
    st = batch.StreamRenderer(ms, sd, cfg.block)
    blocks = [st.step(y[:, b * 256:(b + 1) * 256].contiguous()).clone() for b in range(cfg.ny // 256)]
    streamed = torch.cat(blocks, dim=1)
    assert rel_l2(streamed.cpu().numpy(), offline[:, :cfg.ny].cpu().numpy()) < TOL
    # flushing with zero blocks yields the M-1 tail
    z = torch.zeros((cfg.sources, 256), device="cuda")
    tail = st.step(z).clone()
    assert rel_l2(tail[:, :199].cpu().numpy(), offline[:, cfg.ny:].cpu().numpy()) < TOL
    # strided windows of resident arrays in and out (as the cfg4 tool streams)
    st.reset()
    full = torch.empty((2, cfg.ny), device="cuda")
    for b in range(cfg.ny // 256):
        st.step(y[:, b * 256:(b + 1) * 256], out=full[:, b * 256:(b + 1) * 256])
    assert rel_l2(full.cpu().numpy(), offline[:, :cfg.ny].cpu().numpy()) < TOL
    # reset restarts from silence
    st.reset()
    again = st.step(y[:, :256].contiguous())
    assert rel_l2(again.cpu().numpy(), offline[:, :256].cpu().numpy()) < TOL


def test_time_split_segments_stitch(mods):
    """The multi-GPU split of bench.py --gpus N: segment renders of
    y[t0 - (M-1), t1) give exactly the full render's samples [t0, t1)."""
    batch, _, synth = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("ts", ny=20_000, M=200, K=100, nnz=16, dirs=140, ears=2)
    ms = synth.models(cfg, seed=61)
    y = synth.source(cfg.ny, seed=62)
    br = batch.BatchRenderer(ms)
    full = br.render_all(y).cpu().numpy()
    M, L = cfg.M, cfg.ny + cfg.M - 1
    world = 3
    seg = -(-L // world)
    for r in range(world):
        t0, t1 = min(L, r * seg), min(L, (r + 1) * seg)
        lo = max(0, t0 - (M - 1))
        hi = max(min(cfg.ny, t1), lo + 1)
        part = br.render_all(y[lo:hi]).cpu().numpy()
        got = part[:, :, t0 - lo:t1 - lo]
        ref = full[:, :, t0:t1]
        assert rel_l2(got, ref) < TOL, r
