"""toepnmf kernel module backed by libtoep_b200.so (B200, sm_100a) -- the
INTEGRATION.md section 1 stub, installed by oracle/make_ref_cuda.py into a
scratch copy of the reference as ``toepnmf/engine/_kernels_cuda.py``.

TEST INFRASTRUCTURE: it lets the reference's own engine tests
(pkg/tests/test_engine.py) run against the CUDA kernels through the
reference's plugin seam (pkg/src/toepnmf/engine/__init__.py:35-66).
Same protocol as engine/_kernels.pyx:4-6: (result, macs)."""
import ctypes
import os

import numpy as np
import torch  # device memory + streams only

_L = ctypes.CDLL(os.environ.get("TOEP_LIB_PATH", "libtoep_b200.so"))
_vp, _i64 = ctypes.c_void_p, ctypes.c_int64
_i64p, _fp = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_float)
_L.toep_conv_dense.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64p, _vp]
_L.toep_conv_sparse.argtypes = [_vp, _i64, _i64p, _fp, _i64, _i64, _vp, _i64p, _vp]
_L.toep_fft.argtypes = [_vp, _vp, _i64, ctypes.c_int, _i64p, _vp]
_L.toep_last_error.restype = ctypes.c_char_p


def _check(rc):
    if rc:
        from ..errors import DataError
        raise DataError(_L.toep_last_error().decode())


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def conv_dense(y, taps):
    yd, hd = _dev(y), _dev(taps)
    out = torch.empty(yd.numel() + hd.numel() - 1, device="cuda")
    macs = ctypes.c_int64()
    _check(_L.toep_conv_dense(yd.data_ptr(), yd.numel(), hd.data_ptr(), hd.numel(), out.data_ptr(),
                              ctypes.byref(macs), _stream()))
    return out.cpu().numpy().astype(np.float64), macs.value


def conv_sparse(y, indices, values, length):
    yd = _dev(y)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    val = np.ascontiguousarray(values, dtype=np.float32)
    out = torch.empty(yd.numel() + int(length) - 1, device="cuda")
    macs = ctypes.c_int64()
    _check(_L.toep_conv_sparse(yd.data_ptr(), yd.numel(), idx.ctypes.data_as(_i64p), val.ctypes.data_as(_fp),
                               idx.size, int(length), out.data_ptr(), ctypes.byref(macs), _stream()))
    return out.cpu().numpy().astype(np.float64), macs.value


def fft(data, bitrev, twiddles, inverse):
    d = torch.from_numpy(np.ascontiguousarray(data, np.complex128)).cuda()
    out = torch.empty_like(d)
    macs = ctypes.c_int64()
    _check(_L.toep_fft(d.data_ptr(), out.data_ptr(), d.numel(), int(bool(inverse)), ctypes.byref(macs), _stream()))
    return out.cpu().numpy(), macs.value
