"""Pin the CPU oracle (oracle/toep_oracle.c) before trusting it.

Checked against (1) the golden vectors produced by the reference's own
public API (tests/golden/make_golden.py) and (2) the reference's compiled
Cython kernels (oracle/_ref) on random inputs, when they are built here.
The conv kernels follow the reference loops exactly, so equality is bitwise.
"""
import numpy as np
import pytest

import oracle
from golden_data import golden, rows_of


def test_kat_integer_answers():
    g = golden()
    for mode in ("sparse_direct", "dense_direct"):
        np.testing.assert_array_equal(g["kat_pinned_small_%s" % mode], [3.0, 10.0, 8.0])
        np.testing.assert_array_equal(g["kat_identity_%s" % mode], [3.0, -1.0, 2.0])
    np.testing.assert_array_equal(g["kat_pinned_sparse"], [1, 1, 1, 2, 2, 2])
    assert int(g["kat_pinned_sparse_macs"]) == 2 * 3
    assert int(g["kat_pinned_small_dense_direct_macs"]) == 2 * 2


def test_oracle_dense_bitexact_vs_golden():
    g = golden()
    for i in range(6):
        out, macs = oracle.conv_dense(g["dense_%d_y" % i], g["dense_%d_taps" % i])
        np.testing.assert_array_equal(out, g["dense_%d_out" % i])
        assert macs == g["dense_%d_taps" % i].size * g["dense_%d_y" % i].size


def test_oracle_sparse_bitexact_vs_golden():
    g = golden()
    for i in range(6):
        out, macs = oracle.conv_sparse(g["sparse_%d_y" % i], g["sparse_%d_idx" % i], g["sparse_%d_vals" % i],
                                       int(g["sparse_%d_len" % i]))
        np.testing.assert_array_equal(out, g["sparse_%d_out" % i])
        assert macs == int(g["sparse_%d_macs" % i])


def test_oracle_render_cfg1_bitexact():
    from paper_1502_03162_b200 import synth
    g = golden()
    y = synth.source(44_100, seed=11)
    np.testing.assert_allclose([y.sum(), np.abs(y).sum(), y[:1000].std()], g["cfg1_y_sum"], rtol=0, atol=0)
    out = oracle.render_rows(y, g["cfg1_f"][None], [(g["cfg1_idx"], g["cfg1_vals"])], 100, 1)
    np.testing.assert_array_equal(out[0], g["cfg1_out"])
    # Renderer.counters of the reference: resonance 101*44100, reflection 12*44200, 0 hits, 1 miss
    np.testing.assert_array_equal(g["cfg1_counters"], [101 * 44100, 12 * 44200, 0, 1])


def test_oracle_render_two_ears_bitexact():
    g = golden()
    f = np.stack([g["g2_f_0"], g["g2_f_1"]])
    y = g["g2_y"].astype(np.float64)
    out = oracle.render_rows(y, f, rows_of("g2", 2, 4), 100, 4)
    np.testing.assert_array_equal(out, g["g2_out"])


def test_oracle_render_dense_model():
    g = golden()
    G = g["dense_model_G"]
    rows = [(np.flatnonzero(G[j]), G[j][np.flatnonzero(G[j])]) for j in range(4)]
    out = oracle.render_rows(g["dense_model_y"], g["dense_model_f"][None], rows, 6, 4)
    np.testing.assert_array_equal(out, g["dense_model_out"])


@pytest.mark.parametrize("t0,W", [(0, 1399), (0, 500), (300, 700), (1100, 299)])
def test_oracle_mix_window(t0, W):
    g = golden()
    f = np.stack([g["mx_f_0"], g["mx_f_1"]])
    ys = g["mx_y"].astype(np.float64)
    out = oracle.mix_window(ys, g["mx_dir"], f, rows_of("mx", 2, 9), 100, 9, t0, W, nthreads=3)
    ref = g["mx_out"][:, t0:t0 + W]
    assert np.max(np.abs(out - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_oracle_matches_reference_kernels_random():
    ref = oracle.ref_kernels()
    if ref is None:
        pytest.skip("reference kernels not built (oracle/_ref)")
    rng = np.random.default_rng(99)
    for _ in range(20):
        ny, nt = int(rng.integers(1, 3000)), int(rng.integers(1, 300))
        y, h = rng.standard_normal(ny), rng.standard_normal(nt)
        np.testing.assert_array_equal(oracle.conv_dense(y, h)[0], ref.conv_dense(y, h)[0])
        length = int(rng.integers(1, 400))
        nnz = int(rng.integers(0, min(length, 40) + 1))
        idx = np.sort(rng.choice(length, nnz, replace=False)).astype(np.int64)
        vals = rng.uniform(0.1, 2.0, nnz)
        a, ma = oracle.conv_sparse(y, idx, vals, length)
        b, mb = ref.conv_sparse(y, idx, vals, length)
        np.testing.assert_array_equal(a, b)
        assert ma == mb


def test_cost_model_golden():
    from paper_1502_03162_b200 import engine
    g = golden()
    assert [engine.time_domain_crossover(44100), engine.time_domain_crossover(2205)] == list(g["cost_crossover"])
    assert engine.cost_per_sample_fft(25, 44100) == float(g["cost_fft_25_44100"])
    assert engine.cost_per_sample_fft(1024, 1024) == float(g["cost_fft_1024_1024"])
