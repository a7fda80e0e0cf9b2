"""Drop-in engine API on the GPU: the reference's own engine tests
(pkg/tests/test_engine.py) re-run against the CUDA path.

Integer known-answer tests are exact in fp32; random-property tests carry the
BASELINE tolerance (relative L2 <= 1e-5) instead of the reference's fp64
1e-9..1e-12, because the kernels compute in fp32.
"""
import numpy as np
import pytest

from conftest import TOL, exact_model_data, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng(cuda):
    from paper_1502_03162_b200 import engine
    return engine


def all_mode_outputs(eng, taps, y, **kw):
    return [eng.convolve(eng.ConvPlan(taps, mode, **kw), y) for mode in eng.MODES]


class TestConvolveKAT:
    # pkg/tests/test_engine.py:44-56
    def test_identity_taps(self, eng):
        y = np.array([3.0, -1.0, 2.0])
        for out in all_mode_outputs(eng, np.array([1.0]), y):
            np.testing.assert_allclose(out, y, atol=1e-6)

    def test_pinned_small(self, eng):
        for out in all_mode_outputs(eng, np.array([1.0, 2.0]), np.array([3.0, 4.0])):
            np.testing.assert_allclose(out, [3.0, 10.0, 8.0], atol=1e-5)

    def test_pinned_small_direct_exact(self, eng):
        for mode in ("sparse_direct", "dense_direct"):
            out = eng.convolve(eng.ConvPlan(np.array([1.0, 2.0]), mode), np.array([3.0, 4.0]))
            assert out.dtype == np.float64
            np.testing.assert_array_equal(out, [3.0, 10.0, 8.0])

    def test_pinned_sparse(self, eng):
        from paper_1502_03162_b200 import SparseFilter
        taps = SparseFilter(np.array([0, 3]), np.array([1.0, 2.0]), 4)
        out = eng.convolve(eng.ConvPlan(taps, "sparse_direct"), np.array([1.0, 1.0, 1.0]))
        np.testing.assert_array_equal(out, [1.0, 1.0, 1.0, 2.0, 2.0, 2.0])

    def test_output_length(self, eng):
        rng = np.random.default_rng(2)
        out = eng.convolve(eng.ConvPlan(rng.standard_normal(5), "dense_direct"), rng.standard_normal(11))
        assert out.shape == (15,)

    def test_sparse_taps_in_every_mode(self, eng):
        from paper_1502_03162_b200 import SparseFilter
        rng = np.random.default_rng(0)
        taps = SparseFilter(np.array([1, 4, 7]), rng.uniform(0.5, 1.5, 3), 9)
        y = rng.standard_normal(40)
        expected = np.convolve(y, taps.to_dense())
        for out in all_mode_outputs(eng, taps, y):
            assert rel_l2(out, expected) < TOL

    def test_modes_agree_on_random_pairs(self, eng):
        """pkg/tests/test_engine.py:67-80 incl. the degenerate length 1."""
        rng = np.random.default_rng(1)
        lengths = [(1, 1), (1, 17), (17, 1)] + [(int(rng.integers(1, 200)), int(rng.integers(1, 200)))
                                                  for _ in range(30)]
        for ntaps, ny in lengths:
            taps = rng.standard_normal(ntaps)
            y = rng.standard_normal(ny)
            ref = np.convolve(y, taps)
            for out in all_mode_outputs(eng, taps, y):
                assert out.shape == ref.shape
                assert rel_l2(out, ref) < TOL

    def test_block_size_independence(self, eng):
        rng = np.random.default_rng(4)
        taps = rng.standard_normal(30)
        y = rng.standard_normal(500)
        reference = np.convolve(y, taps)
        for exponent in range(7, 14):
            plan = eng.ConvPlan(taps, "fft_overlap_save", block_size=2 ** exponent)
            assert plan.block_size == 2 ** exponent
            assert rel_l2(eng.convolve(plan, y), reference) < TOL

    def test_validation(self, eng):
        from paper_1502_03162_b200 import DataError
        with pytest.raises(DataError):
            eng.ConvPlan(np.ones(3), "zero_padded")
        with pytest.raises(DataError):
            eng.ConvPlan(np.array([]), "dense_direct")
        with pytest.raises(DataError):
            eng.ConvPlan(np.array([np.inf]), "dense_direct")
        plan = eng.ConvPlan(np.ones(3), "dense_direct")
        with pytest.raises(DataError):
            eng.convolve(plan, np.array([]))
        with pytest.raises(DataError):
            eng.convolve(plan, np.array([np.nan]))

    def test_torch_in_torch_out(self, eng, cuda):
        torch = cuda
        y = torch.randn(1000, device="cuda")
        out = eng.convolve(eng.ConvPlan(np.array([0.5, 0.25]), "dense_direct"), y)
        assert out.is_cuda and out.dtype == torch.float32 and out.numel() == 1001
        ref = np.convolve(y.cpu().numpy().astype(np.float64), [0.5, 0.25])
        assert rel_l2(out.cpu().numpy(), ref) < TOL


class TestMacs:
    # pkg/tests/test_engine.py:127-151
    def test_sparse_macs_exact(self, eng):
        from paper_1502_03162_b200 import SparseFilter
        rng = np.random.default_rng(5)
        taps = SparseFilter(np.array([0, 2, 9]), rng.uniform(0.5, 1.0, 3), 12)
        plan = eng.ConvPlan(taps, "sparse_direct")
        eng.convolve(plan, rng.standard_normal(57))
        assert plan.macs == 3 * 57

    def test_dense_macs_exact(self, eng):
        plan = eng.ConvPlan(np.ones(6), "dense_direct")
        eng.convolve(plan, np.ones(20))
        assert plan.macs == 6 * 20

    def test_macs_accumulate(self, eng):
        plan = eng.ConvPlan(np.ones(4), "dense_direct")
        eng.convolve(plan, np.ones(10))
        eng.convolve(plan, np.ones(10))
        assert plan.macs == 2 * 4 * 10

    def test_fft_macs_positive(self, eng):
        plan = eng.ConvPlan(np.ones(16), "fft_overlap_save")
        eng.convolve(plan, np.ones(100))
        assert plan.macs > 0


class TestRenderer:
    # pkg/tests/test_engine.py:220-281
    @pytest.fixture
    def model(self):
        from paper_1502_03162_b200 import FactorizedModel
        _, f0, G0 = exact_model_data(24, 4, 6, seed=10)
        return FactorizedModel(f0, G0)

    def test_matches_single_stage_convolution(self, eng, model):
        y = np.random.default_rng(11).standard_normal(200)
        for j in range(model.num_directions):
            expected = np.convolve(y, model.reconstruct()[:, j])
            assert rel_l2(eng.render(model, y, j), expected) < TOL

    def test_scaled_impulse_reflection(self, eng):
        from paper_1502_03162_b200 import FactorizedModel
        f = np.array([1.0, -0.5, 0.25])
        model = FactorizedModel(f, np.array([[2.5, 0.0, 0.0, 0.0]]))
        y = np.random.default_rng(12).standard_normal(50)
        got = eng.render(model, y, 0)
        base = np.convolve(y, f)
        np.testing.assert_allclose(got[: base.size], 2.5 * base, rtol=1e-6, atol=1e-6)
        np.testing.assert_array_equal(got[base.size:], 0.0)

    def test_resonance_cache_reused(self, eng, model):
        y = np.random.default_rng(13).standard_normal(150)
        r = eng.Renderer(model)
        r.render(y, 0)
        after_first = r.counters["resonance_macs"]
        assert r.counters["cache_misses"] == 1
        r.render(y, 1)
        assert r.counters["resonance_macs"] == after_first
        assert r.counters["cache_hits"] == 1
        assert r.counters["reflection_macs"] > 0

    def test_new_signal_invalidates_cache(self, eng, model):
        rng = np.random.default_rng(14)
        r = eng.Renderer(model)
        r.render(rng.standard_normal(60), 0)
        r.render(rng.standard_normal(60), 0)
        assert r.counters["cache_misses"] == 2

    def test_direction_range_checked(self, eng, model):
        from paper_1502_03162_b200 import DataError
        with pytest.raises(DataError):
            eng.render(model, np.ones(10), 99)

    def test_fft_mode_renders(self, eng, model):
        y = np.random.default_rng(16).standard_normal(300)
        expected = np.convolve(y, model.reconstruct()[:, 2])
        assert rel_l2(eng.render(model, y, 2, mode="fft_overlap_save"), expected) < TOL


class TestRadix2:
    def test_matches_numpy(self, eng):
        rng = np.random.default_rng(6)
        for n in (1, 2, 8, 64, 256):
            data = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            np.testing.assert_allclose(eng.radix2_fft(data), np.fft.fft(data), atol=1e-10)

    def test_inverse_round_trip(self, eng):
        rng = np.random.default_rng(7)
        data = rng.standard_normal(128) + 1j * rng.standard_normal(128)
        np.testing.assert_allclose(eng.radix2_fft(eng.radix2_fft(data), inverse=True), data, atol=1e-12)


class TestBench:
    def test_row_shape_and_csv(self, eng, tmp_path):
        rows = eng.bench(256, [2, 8], repeats=3)
        assert len(rows) == 2 * len(eng.MODES)
        assert all(r.ns_per_sample_median > 0 and r.backend == "cuda" for r in rows)
        path = str(tmp_path / "bench.csv")
        eng.write_bench_csv(rows, path, include_backend=True)
        lines = open(path).read().splitlines()
        assert lines[0] == eng.BENCH_CSV_HEADER + ",backend"
        assert len(lines) == 1 + len(rows)


class TestFftKernels:
    """fft.cu: complex128 plugin transform across the shared-memory / global
    boundary, and the complex64 overlap-save convolution for every block size
    the reference allows (engine/__init__.py:104-139) up to the global path."""

    @pytest.mark.parametrize("n", [1, 2, 4, 128, 8192, 16384, 1 << 18])
    def test_fft_sizes(self, eng, n):
        rng = np.random.default_rng(n)
        data = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        got = eng.radix2_fft(data)
        ref = np.fft.fft(data)
        assert np.max(np.abs(got - ref)) <= 1e-9 * max(1.0, np.max(np.abs(ref)))
        back = eng.radix2_fft(got, inverse=True)
        assert np.max(np.abs(back - data)) <= 1e-11 * max(1.0, np.max(np.abs(data)))

    def test_fft_in_place_abi(self, eng, cuda):
        from paper_1502_03162_b200 import _lib
        torch = cuda
        for n in (64, 1 << 15):
            x = torch.randn(n, dtype=torch.complex128, device="cuda")
            ref = torch.fft.fft(x)
            y = x.clone()
            assert _lib.fft_c128(y, y, False) == (n // 2) * (n.bit_length() - 1)
            assert float((y - ref).abs().max()) <= 1e-9 * float(ref.abs().max())

    @pytest.mark.parametrize("ntaps,block", [(3, None), (100, None), (100, 128), (200, 1 << 13), (5000, None),
                                             (9000, 1 << 16)])
    def test_overlap_save_blocks(self, eng, ntaps, block):
        rng = np.random.default_rng(ntaps)
        taps = rng.uniform(0.5, 1.5, size=ntaps)
        y = rng.standard_normal(70_000)
        plan = eng.ConvPlan(taps, "fft_overlap_save", block_size=block)
        got = eng.convolve(plan, y)
        assert rel_l2(got, np.convolve(y, taps)) < TOL
