"""The reference's own engine tests, run through the reference's plugin seam
against the CUDA kernels.

oracle/make_ref_cuda.py (run by __graft_entry__.build() where /root/reference
exists) prepares oracle/_ref/pkg_cuda: a copy of the reference package whose
engine (pkg/src/toepnmf/engine/__init__.py:35-66) gains the "cuda" backend --
the ctypes stub over libtoep_b200.so -- as its default, with the fp64
tolerances of pkg/tests/test_engine.py re-set to the fp32 bar (1e-5).  Every
engine test then runs on the GPU: the three modes, the backend agreement and
MAC-count tests against the NumPy backend (:181-205), the renderer cache and
counters, and the bench harness."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "oracle", "_ref", "pkg_cuda")
LIB = os.path.join(ROOT, "paper_1502_03162_b200", "libtoep_b200.so")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.path.join(PKG, "src")
    env["TOEP_LIB_PATH"] = LIB
    env.pop("TOEPNMF_FORCE_PY", None)
    return env


@pytest.fixture(scope="module")
def pkg(cuda):
    if not os.path.isdir(os.path.join(PKG, "tests")):
        pytest.skip("oracle/_ref/pkg_cuda not built (needs /root/reference at build time)")
    return PKG


def test_cuda_is_the_reference_default_backend(pkg):
    out = subprocess.run([sys.executable, "-c", "import toepnmf.engine as e; print(e.DEFAULT_BACKEND, e.available_backends())"],
                         env=_env(), cwd=pkg, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split()[0] == "cuda", out.stdout


def test_reference_engine_suite_on_cuda(pkg):
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "tests/test_engine.py"],
                         env=_env(), cwd=pkg, capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-4000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    assert " passed" in out.stdout and "failed" not in out.stdout.split("\n")[-2], tail
