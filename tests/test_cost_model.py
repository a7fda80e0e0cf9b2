"""The measured B200 cost model (engine.measured_cost_per_sample / measured_crossover)
next to the reference's flop model (engine/__init__.py:278-313).

The table (paper_1502_03162_b200/data/b200_costs.json) is written by
tools/measure_costs.py on a B200: device ns per output sample at the paper's
two signal lengths, per-call for every mode and batched (256 directions in
one fused launch).  These tests run on CPU against the committed table."""
import math

import pytest

from paper_1502_03162_b200 import DataError, engine


def test_table_shape():
    t = engine.measured_cost_table()
    assert set(t["sizes"]) == {"2205", "44100"}
    for n, sizes in t["sizes"].items():
        assert sizes == sorted(sizes) and sizes[0] == 1
        for mode in engine.MODES:
            vals = t["percall"][n][mode]
            assert len(vals) == len(sizes) and all(v > 0 and math.isfinite(v) for v in vals)
        assert len(t["batched"][n]) == len(sizes) and all(v > 0 for v in t["batched"][n])


def test_interpolation_hits_measured_points():
    t = engine.measured_cost_table()
    for n, sizes in t["sizes"].items():
        for mode in engine.MODES:
            for k, v in zip(sizes, t["percall"][n][mode]):
                assert math.isclose(engine.measured_cost_per_sample(mode, k, int(n)), v, rel_tol=1e-9)
        for k, v in zip(sizes, t["batched"][n]):
            assert math.isclose(engine.measured_cost_per_sample("sparse_direct", k, int(n), "batched"), v,
                                rel_tol=1e-9)
    # between points: between the neighbours
    a = engine.measured_cost_per_sample("dense_direct", 100, 44100)
    b = engine.measured_cost_per_sample("dense_direct", 110, 44100)
    c = engine.measured_cost_per_sample("dense_direct", 124, 44100)
    assert min(a, c) <= b <= max(a, c)


@pytest.mark.parametrize("n", [2205, 44100])
@pytest.mark.parametrize("path", ["percall", "batched"])
def test_crossover(n, path):
    t = engine.measured_cost_table()
    top = max(t["sizes"][str(n)])
    c = engine.measured_crossover(n, path)
    assert 0 <= c <= top
    direct = lambda k: engine.measured_cost_per_sample("sparse_direct", k, n, path)
    fft = lambda k: engine.measured_cost_per_sample("fft_overlap_save", k, n, path)
    assert all(direct(k) < fft(k) for k in range(1, c + 1))
    if c < top:
        assert direct(c + 1) >= fft(c + 1)


def test_reference_flop_model_unchanged():
    assert engine.time_domain_crossover(44100) == 124
    assert engine.time_domain_crossover(2205) == 95


def test_bad_arguments():
    with pytest.raises(DataError):
        engine.measured_cost_per_sample("zero_padded", 4, 44100)
    with pytest.raises(DataError):
        engine.measured_cost_per_sample("dense_direct", 0, 44100)
    with pytest.raises(DataError):
        engine.measured_crossover(44100, path="nowhere")
