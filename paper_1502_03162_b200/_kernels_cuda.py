"""CUDA kernel module behind the engine's plugin seam.

Same protocol as the reference kernel modules (pkg/src/toepnmf/engine/
_kernels.pyx:4-6 and _kernels_py.py:3-7): every function returns
``(result, macs)`` where ``macs`` counts the multiply-accumulates of the
reference algorithm.  Inputs may be numpy arrays (result is a float64 numpy
array, as the reference returns) or CUDA tensors (result is a float32 CUDA
tensor, nothing leaves the device).  The arithmetic always runs on the GPU in
fp32 through libtoep_b200.so; there is no host fallback.
"""
from __future__ import annotations

import collections

import numpy as np

from . import _lib


def _dev(x):
    t = _lib.require_cuda()
    if isinstance(x, t.Tensor):
        return x.to(device="cuda", dtype=t.float32).contiguous(), True
    a = np.ascontiguousarray(x, dtype=np.float32)
    return t.from_numpy(a).to("cuda", non_blocking=False), False


def _host(out, was_torch):
    if was_torch:
        return out
    return out.cpu().numpy().astype(np.float64)


def conv_dense(y, taps):
    """Full linear convolution with dense taps (ref: _kernels.pyx:11-25)."""
    t = _lib.require_cuda()
    yd, is_t = _dev(y)
    hd, _ = _dev(taps)
    out = t.empty(yd.numel() + hd.numel() - 1, device="cuda", dtype=t.float32)
    macs = _lib.conv_dense_dev(yd, hd, out)
    return _host(out, is_t), macs


_TABLES = collections.OrderedDict()  # device tap tables of recent tap sets (the engine re-sends a plan's taps)
_TABLES_MAX = 64


def _table(idx, val, length):
    """Device tap table for (indices, values, length), cached by content (LRU).

    The reference kernel accepts offsets in any order and repeated offsets add
    up (_kernels.pyx:38-43); the table holds the merged, sorted form."""
    key = (int(length), idx.tobytes(), val.tobytes())
    tab = _TABLES.get(key)
    if tab is not None:
        _TABLES.move_to_end(key)
        return tab
    if idx.size and (idx.min() < 0 or idx.max() >= length):
        from .errors import DataError
        raise DataError("indices must lie in [0, %d)" % int(length))
    if not np.all(np.isfinite(val)):
        from .errors import DataError
        raise DataError("values must be finite")
    uniq, inv = np.unique(idx, return_inverse=True)
    merged = np.zeros(uniq.size)
    np.add.at(merged, inv, val)
    tab = _lib.Taps([(uniq, merged)], int(length))
    _TABLES[key] = tab
    if len(_TABLES) > _TABLES_MAX:
        _TABLES.popitem(last=False)
    return tab


def conv_sparse(y, indices, values, length):
    """Convolution touching only the listed taps (ref: _kernels.pyx:28-44).

    ``length`` is the dense filter length and fixes the output length even when
    trailing taps are zero.  Offsets may come in any order and repeat (they
    add up), as in the reference; ``macs`` = len(indices) * len(y).
    """
    t = _lib.require_cuda()
    yd, is_t = _dev(y)
    idx = np.ascontiguousarray(indices.cpu() if hasattr(indices, "cpu") else indices, dtype=np.int64).ravel()
    val = np.ascontiguousarray(values.cpu() if hasattr(values, "cpu") else values, dtype=np.float64).ravel()
    if int(length) < 1:
        from .errors import DataError
        raise DataError("filter length must be at least 1")
    out = t.empty(yd.numel() + int(length) - 1, device="cuda", dtype=t.float32)
    _table(idx, val, length).conv(0, yd, out)
    return _host(out, is_t), int(idx.size) * yd.numel()  # _kernels.pyx:43


def fft(data, bitrev, twiddles, inverse):
    """Power-of-two DFT (ref: _kernels.pyx:47-77): radix-2 in complex128 on the GPU (fft.cu).

    ``bitrev``/``twiddles`` are accepted for signature compatibility (the
    kernel derives both); ``macs`` counts radix-2 butterflies, n/2 * log2(n),
    as the reference does.
    """
    t = _lib.require_cuda()
    is_t = isinstance(data, t.Tensor)
    d = data.to("cuda", t.complex128).contiguous() if is_t else \
        t.from_numpy(np.ascontiguousarray(data, np.complex128)).cuda()
    out = t.empty_like(d)
    macs = _lib.fft_c128(d, out, bool(inverse))
    return (out if is_t else out.cpu().numpy()), macs
