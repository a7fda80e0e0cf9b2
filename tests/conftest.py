"""Shared fixtures.  GPU tests are marked ``gpu``; everything else runs on CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtoep_b200.so")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def rel_l2(got, ref) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))


#: BASELINE.json north_star tolerance: relative L2 <= 1e-5 against the reference.
TOL = 1e-5


def exact_model_data(num_taps, num_directions, reflection_length, seed):
    """Same law as the reference fixture (pkg/tests/conftest.py:31-42)."""
    rng = np.random.default_rng(seed)
    f0 = rng.standard_normal(num_taps - reflection_length + 1)
    f0[0] += 3.0
    G0 = rng.uniform(0.1, 1.0, size=(num_directions, reflection_length))
    X = np.column_stack([np.convolve(f0, G0[j]) for j in range(num_directions)])
    return X, f0, G0


@pytest.fixture(scope="session")
def cuda():
    if not has_gpu():
        pytest.skip("no CUDA device")
    import torch
    from paper_1502_03162_b200 import _lib
    _lib.load_library()
    return torch
