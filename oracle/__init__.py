"""CPU oracle for parity checks -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this package.  The product package
(``paper_1502_03162_b200``) never does; it fails loudly without its CUDA
library instead of falling back here.

Two checkers live here:
  * ``liboracle.so`` -- a plain-C fp64 restatement of the reference hot path
    (toep_oracle.c; each routine cites the reference file:line it follows);
  * ``ref_kernels()`` -- the reference's *own* Cython kernels
    (pkg/src/toepnmf/engine/_kernels.pyx) compiled by ``oracle/Makefile`` into
    ``oracle/_ref/`` from the read-only sources (present in the dev container;
    the built .so travels to the GPU box).
The restatement is pinned against the reference kernels and the committed
golden vectors in tests/test_oracle_pin.py.
"""
from __future__ import annotations

import ctypes
import glob
import importlib.machinery
import importlib.util
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(ref: bool = True) -> None:
    """make liboracle.so (and the reference kernels when /root/reference exists)."""
    targets = ["liboracle.so"]
    if ref and os.path.exists("/root/reference/pkg/src/toepnmf/engine/_kernels.pyx"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path)
        L.orc_conv_dense.restype = ctypes.c_int64
        L.orc_conv_dense.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        L.orc_conv_sparse.restype = ctypes.c_int64
        L.orc_conv_sparse.argtypes = [_dp, ctypes.c_int64, _i64p, _dp, ctypes.c_int64, ctypes.c_int64, _dp]
        L.orc_render_rows.restype = ctypes.c_int
        L.orc_render_rows.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      _i64p, _i64p, _dp, ctypes.c_int64, _i32p, ctypes.c_int, _dp,
                                      ctypes.c_int64, ctypes.c_int]
        L.orc_mix_window.restype = ctypes.c_int
        L.orc_mix_window.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _i32p, ctypes.c_int, _dp,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p, _dp,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _dp, ctypes.c_int]
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def conv_dense(y, taps):
    """Reference conv_dense (_kernels.pyx:11-25) in fp64 -> (out, macs)."""
    y, taps = _f64(y), _f64(taps)
    out = np.empty(y.size + taps.size - 1)
    macs = lib().orc_conv_dense(_p(y, _dp), y.size, _p(taps, _dp), taps.size, _p(out, _dp))
    return out, int(macs)


def conv_sparse(y, indices, values, length):
    """Reference conv_sparse (_kernels.pyx:28-44) in fp64 -> (out, macs)."""
    y, values = _f64(y), _f64(values)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    out = np.empty(y.size + int(length) - 1)
    macs = lib().orc_conv_sparse(_p(y, _dp), y.size, _p(idx, _i64p), _p(values, _dp), idx.size, int(length),
                                 _p(out, _dp))
    return out, int(macs)


def _csr(rows_taps):
    """[(indices, values), ...] -> row_ptr, idx, vals (int64/int64/float64)."""
    counts = [len(np.atleast_1d(i)) for i, _ in rows_taps]
    row_ptr = np.zeros(len(rows_taps) + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(counts)
    idx = np.concatenate([np.asarray(i, dtype=np.int64).ravel() for i, _ in rows_taps]) if rows_taps else np.zeros(0, np.int64)
    vals = np.concatenate([np.asarray(v, dtype=np.float64).ravel() for _, v in rows_taps]) if rows_taps else np.zeros(0)
    return row_ptr, np.ascontiguousarray(idx), np.ascontiguousarray(vals)


def render_rows(y, f, rows_taps, K, dirs, rows=None, nthreads=None):
    """Renderer.render (engine/__init__.py:238-260) for ear-major rows.

    f: [ears, lf]; rows_taps: ears*dirs (indices, values) pairs.  Returns
    [len(rows), ny + lf + K - 2] fp64.
    """
    y = _f64(y)
    f = np.atleast_2d(_f64(f))
    ears, lf = f.shape
    row_ptr, idx, vals = _csr(rows_taps)
    if rows is None:
        rows = np.arange(len(rows_taps), dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    L = y.size + lf + K - 2
    out = np.empty((rows.size, L))
    nthreads = nthreads or os.cpu_count() or 1
    rc = lib().orc_render_rows(_p(y, _dp), y.size, _p(f, _dp), lf, ears, dirs, _p(row_ptr, _i64p), _p(idx, _i64p),
                               _p(vals, _dp), K, _p(rows, _i32p), rows.size, _p(out, _dp), L, nthreads)
    assert rc == 0
    return out


def mix_window(y, src_dir, f, rows_taps, K, dirs, t0, W, nthreads=None):
    """sum_s Renderer_e.render(y_s, dir(s))[t0:t0+W] per ear, exact via cropping."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    S, T = y.shape
    f = np.atleast_2d(_f64(f))
    ears, lf = f.shape
    row_ptr, idx, vals = _csr(rows_taps)
    sd = np.ascontiguousarray(src_dir, dtype=np.int32)
    out = np.empty((ears, W))
    nthreads = nthreads or os.cpu_count() or 1
    rc = lib().orc_mix_window(_p(y, _dp), T, T, _p(sd, _i32p), S, _p(f, _dp), lf, ears, dirs,
                              _p(row_ptr, _i64p), _p(idx, _i64p), _p(vals, _dp), K, int(t0), int(W),
                              _p(out, _dp), nthreads)
    assert rc == 0
    return out


def ref_kernels():
    """The reference's own compiled kernel module (oracle/_ref), or None."""
    global _REF
    if _REF is None:
        cands = glob.glob(os.path.join(HERE, "_ref", "_kernels*.so"))
        if not cands:
            return None
        loader = importlib.machinery.ExtensionFileLoader("_kernels", cands[0])
        spec = importlib.util.spec_from_file_location("_kernels", cands[0], loader=loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _REF = mod
    return _REF
