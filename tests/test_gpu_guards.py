"""GPU: no kernel writes outside the buffer it was handed.

compute-sanitizer is not available on the GPU pool, so out-of-bounds stores
are checked with guard bands: every output buffer is a view into a larger
allocation filled with a NaN sentinel (bands before and after the view, row
padding between out_len and the pitch), and after the call the sentinel must
be intact everywhere outside the samples the call owns.  The owned samples
are compared with the oracle so a correct result cannot hide a stray store.
Shapes are picked to end on partial tiles: 133 directions (a partial
128-direction chunk), signal lengths that are not tile multiples.
"""
import numpy as np
import pytest

import oracle
from conftest import TOL, rel_l2

pytestmark = pytest.mark.gpu

GUARD = 1024  # floats before and after each view (16-byte aligned)


@pytest.fixture(scope="module")
def mods(cuda):
    from paper_1502_03162_b200 import batch, synth
    from paper_1502_03162_b200.batch import model_rows
    return batch, synth, model_rows, cuda


def _guarded(torch, shape):
    """(flat buffer, contiguous view of `shape` starting GUARD floats in), NaN-filled."""
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), float("nan"), device="cuda", dtype=torch.float32)
    return buf, buf[GUARD:GUARD + n].view(*shape)


def _bands_intact(buf, n):
    b = buf.cpu().numpy()
    return np.isnan(b[:GUARD]).all() and np.isnan(b[GUARD + n:]).all()


@pytest.mark.parametrize("K,nnz,path,env", [
    (100, 16, "tensor", None),      # k_render_mma (TMA tensor stores, partial last chunk)
    (150, 4, "window", None),       # k_render (bulk stores)
    (100, 16, "window", "0"),       # k_render forced on a K <= 128 filter
    (600, 8, "banded", None),       # k_fir + k_sparse_generic
])
def test_render_stays_in_bounds(mods, monkeypatch, K, nnz, path, env):
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200.synth import Config
    if env is not None:
        monkeypatch.setenv("TOEP_RENDER_MMA", env)
    M = K + 100 if K + 100 > 200 else 200
    cfg = Config("g", ny=5_003, M=M, K=K, nnz=nnz, dirs=133, ears=2)
    ms = synth.models(cfg, seed=K + nnz)
    br = batch.BatchRenderer(ms)
    assert br.native.path() == path
    y = synth.source(cfg.ny, seed=5)
    L = br.out_len(cfg.ny)
    pitch = (L + 3) // 4 * 4 + 12  # 12+ floats of row padding
    buf, out = _guarded(torch, (cfg.ears, cfg.dirs, pitch))
    br.render_all(torch.from_numpy(y.astype(np.float32)).cuda(), out=out)
    torch.cuda.synchronize()
    assert _bands_intact(buf, out.numel())
    host = out.cpu().numpy()
    # the ABI (include/toep_b200.h, toep_renderer_render) may write zeros up to
    # min_pitch (TMA / bulk stores move whole 16-byte units); nothing beyond
    mp = br.native.min_pitch(cfg.ny)
    assert mp == (L + 3) // 4 * 4
    # the recommended pitch (BatchRenderer.alloc) keeps rows on 128-byte lines
    assert br.native.pitch(cfg.ny) == (L + 31) // 32 * 32
    assert br.alloc(cfg.ny).shape[2] == (L + 31) // 32 * 32
    tail = host[:, :, L:mp]
    assert (np.isnan(tail) | (tail == 0)).all(), "non-zero store past out_len"
    assert np.isnan(host[:, :, mp:]).all(), "store into row padding"
    assert not np.isnan(host[:, :, :L]).any(), "owned samples left unwritten"
    f = np.stack([m.resonance_taps for m in ms])
    rows = np.array([0, 127, 128, 132, 133, 265], np.int32)
    ref = oracle.render_rows(y, f, model_rows(ms), cfg.K, cfg.dirs, rows=rows)
    flat = host.reshape(-1, pitch)
    for i, r in enumerate(rows):
        assert rel_l2(flat[r, :L], ref[i]) <= TOL, r


def test_mix_stays_in_bounds(mods):
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("m", ny=7_000, M=200, K=100, nnz=24, dirs=40, ears=2, sources=50)  # z/out lengths 7099/7199
    ms = synth.models(cfg, seed=8)
    sd = np.random.default_rng(8).integers(0, cfg.dirs, size=cfg.sources).astype(np.int32)
    mix = batch.MixRenderer(ms, sd, cfg.ny)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=9)
    zp = (mix.z_len + 3) // 4 * 4 + 8
    zbuf, z = _guarded(torch, (cfg.ears, zp))
    z[:, :mix.z_len] = 0.0  # the partial accumulates into z's owned samples
    mix.partial(y, z=z)
    op = (mix.out_len + 3) // 4 * 4 + 8
    obuf, out = _guarded(torch, (cfg.ears, op))
    res = mix.finish(z, out=out)
    torch.cuda.synchronize()
    assert _bands_intact(zbuf, z.numel()) and _bands_intact(obuf, out.numel())
    zh, oh = z.cpu().numpy(), out.cpu().numpy()
    for h, n in ((zh, mix.z_len), (oh, mix.out_len)):
        r4 = (n + 3) // 4 * 4  # whole 16-byte units past the end may hold zeros
        assert (np.isnan(h[:, n:r4]) | (h[:, n:r4] == 0)).all() and np.isnan(h[:, r4:]).all()
    f = np.stack([m.resonance_taps for m in ms])
    ref = oracle.mix_window(y.cpu().numpy().astype(np.float64), sd, f, model_rows(ms), cfg.K, cfg.dirs, 0,
                            mix.out_len)
    got = res.cpu().numpy()
    for e in range(cfg.ears):
        assert rel_l2(got[e], ref[e]) <= TOL


@pytest.mark.parametrize("kernel", ["cluster", "ticketed"])
def test_stream_stays_in_bounds(mods, monkeypatch, kernel):
    monkeypatch.setenv("TOEP_STREAM_CLUSTER", "1" if kernel == "cluster" else "0")
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("s", ny=4 * 96, M=200, K=100, nnz=16, dirs=30, ears=2, sources=20, block=96)
    ms = synth.models(cfg, seed=12)
    sd = np.random.default_rng(12).integers(0, cfg.dirs, size=cfg.sources).astype(np.int32)
    st = batch.StreamRenderer(ms, sd, cfg.block)
    y = synth.device_sources(cfg.sources, cfg.ny, seed=13)
    pitch = cfg.block + 8
    buf, rows = _guarded(torch, (cfg.ears, pitch))
    out = rows[:, :cfg.block]  # [ears, B] with unit column stride, row pitch B + 8
    got = []
    for b in range(cfg.ny // cfg.block):
        st.step(y[:, b * cfg.block:(b + 1) * cfg.block].contiguous(), out=out)
        torch.cuda.synchronize()
        assert _bands_intact(buf, rows.numel())
        assert np.isnan(rows.cpu().numpy()[:, cfg.block:]).all()
        got.append(out.cpu().numpy().copy())
    got = np.concatenate(got, axis=1)
    f = np.stack([m.resonance_taps for m in ms])
    ref = oracle.mix_window(y.cpu().numpy().astype(np.float64), sd, f, model_rows(ms), cfg.K, cfg.dirs, 0,
                            cfg.ny)
    for e in range(cfg.ears):
        assert rel_l2(got[e], ref[e]) <= TOL


def test_fft_conv_stays_in_bounds(mods):
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200 import _lib
    rng = np.random.default_rng(21)
    taps = rng.standard_normal(300).astype(np.float32)
    y = rng.standard_normal(10_007).astype(np.float32)
    n = 1024
    spec = _lib.fft_spectrum(torch.from_numpy(taps).cuda(), n)
    L = y.size + taps.size - 1
    buf, out = _guarded(torch, ((L + 3) // 4 * 4,))
    _lib.fft_conv(torch.from_numpy(y).cuda(), spec, n, taps.size, out)
    torch.cuda.synchronize()
    assert _bands_intact(buf, out.numel())
    ref = np.convolve(y.astype(np.float64), taps.astype(np.float64))
    assert rel_l2(out[:L].cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("ntaps", [1, 5, 101, 600])
def test_conv_dense_exact_length(mods, ntaps):
    """toep_conv_dense writes exactly ny + ntaps - 1 samples (the caller may size out to that)."""
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200 import _lib
    rng = np.random.default_rng(ntaps)
    y = rng.standard_normal(3_001).astype(np.float32)
    taps = rng.standard_normal(ntaps).astype(np.float32)
    L = y.size + ntaps - 1
    buf, out = _guarded(torch, (L,))
    _lib.conv_dense_dev(torch.from_numpy(y).cuda(), torch.from_numpy(taps).cuda(), out)
    torch.cuda.synchronize()
    assert _bands_intact(buf, L)
    assert rel_l2(out.cpu().numpy(), np.convolve(y.astype(np.float64), taps.astype(np.float64))) <= TOL


@pytest.mark.parametrize("K,nnz", [(100, 16), (150, 4), (600, 8)])
def test_conv_sparse_exact_length(mods, K, nnz):
    """toep_conv_sparse writes exactly ny + K - 1 samples on each of its kernels."""
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200 import _lib
    rng = np.random.default_rng(K + nnz)
    y = rng.standard_normal(3_001).astype(np.float32)
    idx = np.sort(rng.choice(K, size=nnz, replace=False)).astype(np.int64)
    val = (np.abs(rng.standard_normal(nnz)) + 0.1).astype(np.float32)
    L = y.size + K - 1
    buf, out = _guarded(torch, (L,))
    _lib.conv_sparse_dev(torch.from_numpy(y).cuda(), idx, val, K, out)
    torch.cuda.synchronize()
    assert _bands_intact(buf, L)
    dense = np.zeros(K)
    dense[idx] = val
    assert rel_l2(out.cpu().numpy(), np.convolve(y.astype(np.float64), dense)) <= TOL


def test_render_long_signal_two_launches_stay_in_bounds(mods):
    """Long signals add the fill launch (its own tile range of every row): both stay inside the rows."""
    batch, synth, model_rows, torch = mods
    from paper_1502_03162_b200.synth import Config
    cfg = Config("L", ny=300_003, M=200, K=100, nnz=16, dirs=9, ears=2)
    ms = synth.models(cfg, seed=77)
    br = batch.BatchRenderer(ms)
    assert br.native.path() == "tensor"
    y = synth.source(cfg.ny, seed=78)
    L = br.out_len(cfg.ny)
    mp = br.native.min_pitch(cfg.ny)
    pitch = mp + 8
    buf, out = _guarded(torch, (cfg.ears, cfg.dirs, pitch))
    br.render_all(torch.from_numpy(y.astype(np.float32)).cuda(), out=out)
    torch.cuda.synchronize()
    assert _bands_intact(buf, out.numel())
    host = out.cpu().numpy()
    tail = host[:, :, L:mp]
    assert (np.isnan(tail) | (tail == 0)).all() and np.isnan(host[:, :, mp:]).all()
    assert not np.isnan(host[:, :, :L]).any()
    f = np.stack([m.resonance_taps for m in ms])
    rows = np.array([0, 8, 9, 17], np.int32)
    ref = oracle.render_rows(y, f, model_rows(ms), cfg.K, cfg.dirs, rows=rows)
    flat = host.reshape(-1, pitch)
    for i, r in enumerate(rows):
        assert rel_l2(flat[r, :L], ref[i]) <= TOL, r
