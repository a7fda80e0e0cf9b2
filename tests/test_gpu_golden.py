"""CUDA path against the golden vectors recorded from the reference's own
public API (tests/golden/make_golden.py).  Tolerance: relative L2 <= 1e-5
per channel (BASELINE north_star); integer known answers are exact."""
import numpy as np
import pytest

from conftest import TOL, rel_l2
from golden_data import golden, rows_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk(cuda):
    from paper_1502_03162_b200 import FactorizedModel, SparseFilter, batch, engine, synth
    return FactorizedModel, SparseFilter, batch, engine, synth


def test_kats_exact(pk):
    _, SparseFilter, _, engine, _ = pk
    g = golden()
    for name, taps, y in (("identity", [1.0], [3.0, -1.0, 2.0]), ("pinned_small", [1.0, 2.0], [3.0, 4.0])):
        for mode in ("sparse_direct", "dense_direct"):
            plan = engine.ConvPlan(np.array(taps), mode)
            np.testing.assert_array_equal(engine.convolve(plan, np.array(y)), g["kat_%s_%s" % (name, mode)])
            assert plan.macs == int(g["kat_%s_%s_macs" % (name, mode)])
    plan = engine.ConvPlan(SparseFilter(np.array([0, 3]), np.array([1.0, 2.0]), 4), "sparse_direct")
    np.testing.assert_array_equal(engine.convolve(plan, np.ones(3)), g["kat_pinned_sparse"])
    assert plan.macs == int(g["kat_pinned_sparse_macs"])


def test_plugin_cases(pk):
    _, SparseFilter, _, engine, _ = pk
    g = golden()
    for i in range(6):
        out = engine.convolve(engine.ConvPlan(g["dense_%d_taps" % i], "dense_direct"), g["dense_%d_y" % i])
        assert out.shape == g["dense_%d_out" % i].shape and rel_l2(out, g["dense_%d_out" % i]) < TOL
    for i in range(6):
        sf = SparseFilter(g["sparse_%d_idx" % i], g["sparse_%d_vals" % i], int(g["sparse_%d_len" % i]))
        plan = engine.ConvPlan(sf, "sparse_direct")
        out = engine.convolve(plan, g["sparse_%d_y" % i])
        assert out.shape == g["sparse_%d_out" % i].shape and rel_l2(out, g["sparse_%d_out" % i]) < TOL
        assert plan.macs == int(g["sparse_%d_macs" % i])


def test_cfg1_golden(pk):
    FactorizedModel, SparseFilter, batch, engine, synth = pk
    g = golden()
    y = synth.source(44_100, seed=11)
    m = FactorizedModel(g["cfg1_f"], [SparseFilter(g["cfg1_idx"], g["cfg1_vals"], 100)])
    r = engine.Renderer(m)
    out = r.render(y, 0)
    assert out.shape == g["cfg1_out"].shape and rel_l2(out, g["cfg1_out"]) < TOL
    c = r.counters
    np.testing.assert_array_equal([c["resonance_macs"], c["reflection_macs"], c["cache_hits"], c["cache_misses"]],
                                  g["cfg1_counters"])
    fused = batch.BatchRenderer([m]).render_all(y)[0, 0].cpu().numpy()
    assert rel_l2(fused, g["cfg1_out"]) < TOL


def test_two_ears_golden(pk):
    FactorizedModel, SparseFilter, batch, engine, _ = pk
    g = golden()
    y = g["g2_y"].astype(np.float64)
    rows = rows_of("g2", 2, 4)
    ms = [FactorizedModel(g["g2_f_%d" % e], [SparseFilter(i, v, 100) for i, v in rows[4 * e:4 * e + 4]])
          for e in range(2)]
    out = batch.BatchRenderer(ms).render_all(y).reshape(8, -1).cpu().numpy()
    for i in range(8):
        assert rel_l2(out[i], g["g2_out"][i]) < TOL
    for e in range(2):  # per-call drop-in path + counters of the reference Renderer
        r = engine.Renderer(ms[e])
        for d in range(4):
            assert rel_l2(r.render(y, d), g["g2_out"][4 * e + d]) < TOL
        c = r.counters
        np.testing.assert_array_equal([c["resonance_macs"], c["reflection_macs"], c["cache_hits"],
                                       c["cache_misses"]], g["g2_counters_%d" % e])


def test_dense_model_golden(pk):
    FactorizedModel, _, batch, engine, _ = pk
    g = golden()
    m = FactorizedModel(g["dense_model_f"], g["dense_model_G"])
    for j in range(4):
        assert rel_l2(engine.render(m, g["dense_model_y"], j), g["dense_model_out"][j]) < TOL
    out = batch.BatchRenderer([m]).render_all(g["dense_model_y"])[0].cpu().numpy()
    for j in range(4):
        assert rel_l2(out[j], g["dense_model_out"][j]) < TOL


def test_mix_golden(pk, cuda):
    FactorizedModel, SparseFilter, batch, _, _ = pk
    torch = cuda
    g = golden()
    rows = rows_of("mx", 2, 9)
    ms = [FactorizedModel(g["mx_f_%d" % e], [SparseFilter(i, v, 100) for i, v in rows[9 * e:9 * e + 9]])
          for e in range(2)]
    y = torch.from_numpy(g["mx_y"]).cuda()
    out = batch.MixRenderer(ms, g["mx_dir"], y.shape[1]).render(y).cpu().numpy()
    for e in range(2):
        assert rel_l2(out[e], g["mx_out"][e]) < TOL
