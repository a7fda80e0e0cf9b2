"""Host-side behaviour of the drop-in API that needs no GPU: validation,
plan bookkeeping, the cost model, bench CSV format, synthetic input laws,
source partitioning -- and the no-fallback rule (compute without the CUDA
path fails loudly instead of running on the CPU)."""
import math

import numpy as np
import pytest

from conftest import has_gpu
from paper_1502_03162_b200 import DataError, FactorizedModel, Signal, SparseFilter, engine, synth
from paper_1502_03162_b200 import dist as tdist


class TestPlans:
    def test_modes_and_backends(self):
        assert engine.MODES == ("sparse_direct", "dense_direct", "fft_overlap_save")
        assert engine.available_backends() == ("cuda",)
        assert engine.DEFAULT_BACKEND == "cuda"

    def test_unknown_backend_rejected(self):
        with pytest.raises(DataError):
            engine.ConvPlan(np.ones(3), "dense_direct", backend="fortran")
        with pytest.raises(DataError):
            engine.ConvPlan(np.ones(3), "dense_direct", backend="python")  # no NumPy fallback
        engine.ConvPlan(np.ones(3), "dense_direct", backend="compiled")  # alias of cuda

    def test_validation(self):
        with pytest.raises(DataError):
            engine.ConvPlan(np.ones(3), "zero_padded")
        with pytest.raises(DataError):
            engine.ConvPlan(np.array([]), "dense_direct")
        with pytest.raises(DataError):
            engine.ConvPlan(np.array([np.inf]), "dense_direct")
        with pytest.raises(DataError):
            engine.ConvPlan(np.ones((2, 2)), "dense_direct")

    def test_block_sizes(self):
        assert engine.ConvPlan(np.ones(30), "fft_overlap_save").block_size == 128
        for e in range(7, 14):
            assert engine.ConvPlan(np.ones(30), "fft_overlap_save", block_size=2 ** e).block_size == 2 ** e
        assert engine.ConvPlan(np.ones(30), "fft_overlap_save", block_size=100).block_size == 128
        with pytest.raises(DataError):
            engine.ConvPlan(np.ones(30), "fft_overlap_save", block_size=16)
        assert engine.ConvPlan(np.ones(30), "dense_direct").block_size is None

    def test_dense_sparse_views(self):
        sf = SparseFilter(np.array([1, 4]), np.array([0.5, 2.0]), 6)
        p = engine.ConvPlan(sf, "dense_direct")
        np.testing.assert_array_equal(p.dense_taps(), [0, 0.5, 0, 0, 2.0, 0])
        q = engine.ConvPlan(np.array([0.0, 3.0, 0.0, 1.0]), "sparse_direct")
        idx, vals, length = q.sparse_parts()
        np.testing.assert_array_equal(idx, [1, 3])
        np.testing.assert_array_equal(vals, [3.0, 1.0])
        assert length == 4 and q.taps_length == 4

    def test_renderer_direction_check_before_compute(self):
        m = FactorizedModel(np.array([1.0, 0.5]), np.array([[1.0, 0.0], [0.0, 2.0]]))
        with pytest.raises(DataError):
            engine.Renderer(m).render(np.ones(4), 2)
        with pytest.raises(DataError):
            engine.Renderer(m, mode="bogus")

    @pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
    def test_no_cpu_fallback(self):
        from paper_1502_03162_b200._lib import NativeUnavailable
        with pytest.raises(NativeUnavailable):
            engine.convolve(engine.ConvPlan(np.ones(3), "dense_direct"), np.ones(5))
        from paper_1502_03162_b200 import batch
        with pytest.raises(NativeUnavailable):
            batch.BatchRenderer(synth.models(synth.Config("x", 10, 20, 10, 2, 2, 1), 0)).render_all(np.ones(10))


class TestTypes:
    def test_sparse_filter_rules(self):
        with pytest.raises(DataError):
            SparseFilter(np.array([2, 1]), np.array([1.0, 1.0]), 4)
        with pytest.raises(DataError):
            SparseFilter(np.array([0, 4]), np.array([1.0, 1.0]), 4)
        with pytest.raises(DataError):
            SparseFilter(np.array([0]), np.array([0.0]), 4)
        with pytest.raises(DataError):
            SparseFilter(np.array([0]), np.array([1.0]), 0)
        empty = SparseFilter(np.array([], dtype=np.int64), np.array([]), 5)
        assert empty.nnze == 0 and np.all(empty.to_dense() == 0)

    def test_model_properties(self):
        m = FactorizedModel(np.ones(3), [SparseFilter(np.array([0]), np.array([1.0]), 4)] * 2)
        assert m.is_sparse and m.num_directions == 2 and m.reflection_length == 4 and m.num_taps == 6
        with pytest.raises(DataError):
            FactorizedModel(np.ones(3), np.array([[-1.0, 0.0]]))

    def test_signal(self):
        with pytest.raises(DataError):
            Signal(np.array([np.nan]), 48000.0)
        with pytest.raises(DataError):
            Signal(np.ones(3), 0.0)


class TestCostModel:
    def test_pinned(self):
        assert engine.cost_per_sample_time_domain(25, 44100) == 25.0
        assert engine.cost_per_sample_time_domain(10, 5) == 5.0
        n = 1024
        assert math.isclose(engine.cost_per_sample_fft(n, n), engine.FFT_COST_FACTOR * (n * math.log2(n) + n),
                            rel_tol=1e-12)
        assert engine.cost_per_sample_fft_real_adjusted(25, 44100) == 3.0 * engine.cost_per_sample_fft(25, 44100)
        with pytest.raises(DataError):
            engine.cost_per_sample_fft(10, 5)
        with pytest.raises(DataError):
            engine.cost_per_sample_time_domain(0, 10)

    def test_crossover(self):
        assert engine.time_domain_crossover(44100) == 124
        assert engine.time_domain_crossover(2205) == 95

    def test_bench_rejects_bad_args(self):
        with pytest.raises(DataError):
            engine.bench(128, [2], repeats=2)
        with pytest.raises(DataError):
            engine.bench(0, [2])
        with pytest.raises(DataError):
            engine.bench(16, [])

    def test_csv_writer(self, tmp_path):
        rows = [engine.BenchRow("dense_direct", 100, 4, 0, 1.5, 4.0, "cuda")]
        p = str(tmp_path / "b.csv")
        engine.write_bench_csv(rows, p)
        assert open(p).read().splitlines() == [engine.BENCH_CSV_HEADER, "dense_direct,100,4,0,1.5,4"]
        engine.write_bench_csv(rows, p, include_backend=True)
        assert open(p).read().splitlines()[1].endswith(",cuda")


class TestSynthAndPartition:
    def test_laws(self):
        cfg = synth.CONFIGS["cfg2"]
        ms = synth.models(synth.Config("t", 100, 200, 100, 16, 20, 2), seed=4)
        assert len(ms) == 2
        for m in ms:
            assert m.resonance_taps.size == 101
            assert abs(np.linalg.norm(m.resonance_taps) - 1.0) < 1e-6
            for r in m.reflections:
                assert r.indices.size == 16 and np.all(np.diff(r.indices) > 0) and np.all(r.values > 0)
                assert r.values.dtype == np.float64 and np.all(r.values == r.values.astype(np.float32))
        assert cfg.lf == 101 and cfg.M == 200
        pts = synth.cfg3_points()
        assert ("cfg3_K50_nnz64" not in [p.name for p in pts]) and len(pts) == 17

    @pytest.mark.parametrize("S,world", [(4096, 1), (4096, 8), (10, 3), (5, 8)])
    def test_partition_covers_each_source_once(self, S, world):
        seen = []
        for r in range(world):
            s0, n = tdist.partition(S, world, r)
            seen.extend(range(s0, s0 + n))
        assert seen == list(range(S))
        sizes = [tdist.partition(S, world, r)[1] for r in range(world)]
        assert max(sizes) - min(sizes) <= 1


def test_partition_by_direction():
    """Every direction's sources on one rank, balanced mix work (sources +
    DIRECTION_COST x distinct directions), each rank touching ~1/N of the
    directions (the mix's tap work)."""
    sd = synth.source_directions(4096, 1250, seed=5)
    for world in (1, 2, 3, 8):
        parts = tdist.partition_by_direction(sd, world)
        assert len(parts) == world
        allidx = np.concatenate(parts)
        assert sorted(allidx.tolist()) == list(range(4096))
        dirs = [set(sd[p].tolist()) for p in parts]
        cost = [len(p) + tdist.DIRECTION_COST * len(d) for p, d in zip(parts, dirs)]
        for i in range(world):
            assert all(not (dirs[i] & dirs[j]) for j in range(i + 1, world))
            assert abs(len(parts[i]) - 4096 / world) <= 0.05 * 4096 / world + 8
            assert abs(cost[i] - sum(cost) / world) <= 0.01 * sum(cost) / world + 8
        assert max(len(d) for d in dirs) <= 1.2 * len(set(sd.tolist())) / world
    sd2 = np.zeros(10, np.int32)  # one direction: kept whole without splitting, split otherwise
    parts = tdist.partition_by_direction(sd2, 4, split=False)
    assert sorted(len(p) for p in parts) == [0, 0, 0, 10]
    parts = tdist.partition_by_direction(sd2, 4)
    assert sorted(len(p) for p in parts) == [2, 2, 3, 3]
