"""GPU parity at BASELINE size for the mixdown configs (4 streaming, 5 sharded
mixdown) and the config-3 sweep at the full 1,250 directions.

The oracle is the reference composition sum_s Renderer_e.render(y_s, dir(s))
(pkg/src/toepnmf/engine/__init__.py:238-260) in fp64, evaluated on exact
windows: output samples [t0, t0+W) depend only on y[t0-(M-1), t0+W)
(oracle.mix_window crops).  Bar: relative L2 <= 1e-5 per ear (north_star).
Size-independent identity on every output sample: the sum of a full linear
convolution is the product of the operand sums, so
sum_t out_e[t] = sum(f_e) * sum_s sum(y_s) * sum(g_{e,dir(s)}).
"""
import numpy as np
import pytest

import oracle
from conftest import TOL, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods(cuda):
    from paper_1502_03162_b200 import batch, dist, synth
    from paper_1502_03162_b200.batch import model_rows
    return batch, dist, synth, model_rows


def _windows_vs_oracle(y, out, ms, sd, K, dirs, T, windows, model_rows):
    f = np.stack([m.resonance_taps for m in ms])
    rows = model_rows(ms)
    worst = 0.0
    for t0, W in windows:
        W = min(W, T + 199 - t0)
        lo = max(0, t0 - 199)
        yc = y[:, lo:min(T, t0 + W)].double().cpu().numpy()
        ref = oracle.mix_window(yc, sd, f, rows, K, dirs, t0 - lo, W)
        got = out[:, t0:t0 + W].double().cpu().numpy()
        for e in range(len(ms)):
            err = rel_l2(got[e], ref[e])
            worst = max(worst, err)
            assert err < TOL, (t0, e, err)
    return worst


def _sum_identity(y, out, ms, sd):
    """sum_t out_e = sum(f_e) * sum_s sum(y_s) * sum(g_{e,d(s)}) for every ear."""
    sy = y.double().sum(dim=1).cpu().numpy()
    for e, m in enumerate(ms):
        gs = np.array([np.sum(r.values) for r in m.reflections])
        want = float(np.sum(m.resonance_taps)) * float(np.sum(sy * gs[sd]))
        got = float(out[e].double().sum().item())
        l1 = float(out[e].double().abs().sum().item())
        assert abs(got - want) <= 1e-6 * l1, (e, got, want)


def test_cfg5_full_size(mods, cuda):
    """Config 5 at BASELINE size (4,096 sources x 2,880,000 samples, nnz 24), the
    bench's seeds; windows at the start, tile seams, past source row 2^31/T,
    and the final tail."""
    batch, _, synth, model_rows = mods
    torch = cuda
    cfg = synth.CONFIGS["cfg5"]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    T = cfg.ny
    y = synth.device_sources_indexed(np.arange(cfg.sources), T, seed=1000)
    mix = batch.MixRenderer(ms, sd, T)
    assert mix.path == "tensor"
    out = mix.render(y)
    torch.cuda.synchronize()
    assert mix.path == "tensor"  # the plan fitted (no fallback)
    assert out.shape == (2, T + 199)
    assert bool(torch.isfinite(out).all())
    windows = [(0, 2048), (256 * 5625 - 100, 700), (2048 * 700 - 5, 1200), (1_000_003, 1500),
               (T + 199 - 2048, 2048)]
    _windows_vs_oracle(y, out, ms, sd, cfg.K, cfg.dirs, T, windows, model_rows)
    _sum_identity(y, out, ms, sd)


def test_cfg5_shards_add_up(mods, cuda):
    """The multi-GPU contract on one GPU: the direction partition's per-rank
    partial mixes (dist.MixShard, world 2 and 8) sum to the one-GPU partial,
    and f on the summed partial matches the oracle (reduced T)."""
    batch, dist, synth, model_rows = mods
    torch = cuda
    cfg = synth.CONFIGS["cfg5"]
    ms = synth.models(cfg, seed=5)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=5)
    T = 120_000
    y = synth.device_sources_indexed(np.arange(cfg.sources), T, seed=1000)
    whole = batch.MixRenderer(ms, sd, T)
    zw = whole.partial(y)[:, :whole.z_len].double()
    for world in (2, 8):
        acc = None
        for rank in range(world):
            sh = dist.MixShard(ms, sd, T, world=world, rank=rank)
            ys = synth.device_sources_indexed(sh.sources, T, seed=1000)
            # rows drawn per global index equal the one-GPU rows
            assert torch.equal(ys[:3], y[torch.as_tensor(sh.sources[:3], device="cuda")])
            z = sh.partial(ys)[:, :whole.z_len].double()
            acc = z if acc is None else acc + z
        assert rel_l2(acc.cpu().numpy(), zw.cpu().numpy()) < TOL
        out = whole.finish(acc.float().contiguous())
        _windows_vs_oracle(y, out, ms, sd, cfg.K, cfg.dirs, T, [(0, 1500), (T - 1000, 1199)], model_rows)


def test_cfg4_stream_full_size(mods, cuda):
    """Config 4 at BASELINE size: 512 sources x 60 s streamed in 11,250 blocks of
    256 (one CUDA graph), compared directly with the oracle on windows of the
    concatenated blocks, plus the flushed tail."""
    batch, _, synth, model_rows = mods
    torch = cuda
    cfg = synth.CONFIGS["cfg4"]
    B = cfg.block
    T = cfg.ny
    ms = synth.models(cfg, seed=4)
    sd = synth.source_directions(cfg.sources, cfg.dirs, seed=4)
    y = synth.device_sources_indexed(np.arange(cfg.sources), T, seed=44)
    st = batch.StreamRenderer(ms, sd, B)
    out = torch.empty((cfg.ears, T + B), device="cuda")
    g = st.capture(y, out, T // B)
    st.reset()
    g.replay()
    # flush: one block of silence yields the M-1 tail
    zero = torch.zeros((cfg.sources, B), device="cuda")
    st.step(zero, out=out[:, T:T + B])
    torch.cuda.synchronize()
    full = out[:, :T + 199]
    windows = [(0, 1024), (B * 5000 - 77, 900), (1_440_007, 1000), (T - 1024, 1024 + 199)]
    _windows_vs_oracle(y, full, ms, sd, cfg.K, cfg.dirs, T, windows, model_rows)
    _sum_identity(y, full, ms, sd)


@pytest.mark.parametrize("K,nnz", [(50, 8), (50, 16), (50, 32), (100, 16), (150, 16), (150, 32)])
def test_cfg3_full_directions(mods, cuda, K, nnz):
    """Config-3 points at the full 1,250 directions x 2 ears (441,000 samples):
    oracle rows across both ears and the row-sum identity on all 2,500 rows."""
    batch, _, synth, _ = mods
    torch = cuda
    from paper_1502_03162_b200.synth import Config
    cfg = Config("p", ny=441_000, M=200, K=K, nnz=nnz, dirs=1250, ears=2)
    ms = synth.models(cfg, seed=K * 1000 + nnz)
    y = synth.source(cfg.ny, seed=3)
    br = batch.BatchRenderer(ms)
    out = br.render_all(y)
    rows = [0, 311, 1249, 1250, 1999, 2499]
    f = np.stack([m.resonance_taps for m in ms])
    from paper_1502_03162_b200.batch import model_rows
    ref = oracle.render_rows(y, f, model_rows(ms), K, cfg.dirs, rows=np.asarray(rows, np.int32))
    got = out.reshape(-1, out.shape[-1])[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    for i in range(len(rows)):
        assert rel_l2(got[i], ref[i]) < TOL, rows[i]
    sy = float(np.sum(y))
    sums = out.double().sum(dim=-1).cpu().numpy()
    l1 = out.double().abs().sum(dim=-1).cpu().numpy()
    for e, m in enumerate(ms):
        want = sy * float(np.sum(m.resonance_taps)) * np.array([np.sum(r.values) for r in m.reflections])
        assert np.all(np.abs(sums[e] - want) <= 1e-6 * l1[e] + 1e-9)
