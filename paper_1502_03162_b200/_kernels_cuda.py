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


def conv_sparse(y, indices, values, length):
    """Convolution touching only the listed taps (ref: _kernels.pyx:28-44).

    ``length`` is the dense filter length and fixes the output length even when
    trailing taps are zero.
    """
    t = _lib.require_cuda()
    yd, is_t = _dev(y)
    idx = np.asarray(indices.cpu() if hasattr(indices, "cpu") else indices, dtype=np.int64)
    val = np.asarray(values.cpu() if hasattr(values, "cpu") else values, dtype=np.float32)
    out = t.empty(yd.numel() + int(length) - 1, device="cuda", dtype=t.float32)
    macs = _lib.conv_sparse_dev(yd, idx, val, int(length), out)
    return _host(out, is_t), macs


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
