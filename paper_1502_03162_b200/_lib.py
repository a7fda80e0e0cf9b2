"""ctypes binding of the C ABI in include/toep_b200.h (libtoep_b200.so).

This is the only place the product touches native code.  There is no CPU or
pure-Python fallback: if the library or a CUDA device is missing, every entry
point raises :class:`NativeUnavailable`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DataError

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOEP_LIB") or os.path.join(PKG_DIR, "libtoep_b200.so")  # TOEP_LIB: experiment builds

TOEP_OK, TOEP_ERR_INVALID, TOEP_ERR_CUDA, TOEP_ERR_NOMEM, TOEP_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

#: every function declared in include/toep_b200.h
EXPORTS = (
    "toep_last_error", "toep_abi_version", "toep_sm_count",
    "toep_conv_dense", "toep_conv_sparse", "toep_fft", "toep_fft_spectrum", "toep_fft_conv",
    "toep_taps_create", "toep_taps_destroy", "toep_taps_info", "toep_taps_conv",
    "toep_renderer_create", "toep_renderer_destroy", "toep_renderer_out_len", "toep_renderer_min_pitch",
    "toep_renderer_pitch",
    "toep_renderer_render", "toep_renderer_reflect", "toep_renderer_check", "toep_renderer_path",
    "toep_renderer_kernels",
    "toep_mixer_create", "toep_mixer_destroy", "toep_mixer_z_len", "toep_mixer_out_len",
    "toep_mixer_partial", "toep_mixer_finish", "toep_mixer_path", "toep_mixer_kernels",
    "toep_streamer_create", "toep_streamer_destroy", "toep_streamer_reset", "toep_streamer_step",
)


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is not available (no fallback exists)."""


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the C ABI."""


_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_fp = ctypes.POINTER(ctypes.c_float)


def load_library(path: str = LIB_PATH):
    """dlopen libtoep_b200.so and declare the C signatures (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            "libtoep_b200.so is not built (run __graft_entry__.build() or "
            "python -m paper_1502_03162_b200._build); there is no CPU fallback")
    L = ctypes.CDLL(path)
    sig = {
        "toep_last_error": (ctypes.c_char_p, []),
        "toep_abi_version": (ctypes.c_int, []),
        "toep_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
        "toep_conv_dense": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64p, _vp]),
        "toep_conv_sparse": (ctypes.c_int, [_vp, _i64, _i64p, _fp, _i64, _i64, _vp, _i64p, _vp]),
        "toep_fft": (ctypes.c_int, [_vp, _vp, _i64, ctypes.c_int, ctypes.POINTER(_i64), _vp]),
        "toep_fft_spectrum": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp]),
        "toep_fft_conv": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i64, _vp, _vp]),
        "toep_taps_create": (ctypes.c_int, [_i32, _i32, _i64p, _i64p, _fp, ctypes.POINTER(_vp)]),
        "toep_taps_destroy": (ctypes.c_int, [_vp]),
        "toep_taps_info": (ctypes.c_int, [_vp, _i32p, _i32p, _i32p, _i64p]),
        "toep_taps_conv": (ctypes.c_int, [_vp, _i32, _vp, _i64, _vp, _vp]),
        "toep_renderer_create": (ctypes.c_int, [_fp, _i32, _i32, _vp, _i32, ctypes.POINTER(_vp)]),
        "toep_renderer_destroy": (ctypes.c_int, [_vp]),
        "toep_renderer_out_len": (_i64, [_vp, _i64]),
        "toep_renderer_min_pitch": (_i64, [_vp, _i64]),
        "toep_renderer_pitch": (_i64, [_vp, _i64]),
        "toep_renderer_render": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _vp]),
        "toep_renderer_reflect": (ctypes.c_int, [_vp, _i32, _vp, _i64, _vp, _i64, _vp]),
        "toep_renderer_check": (ctypes.c_int, [_vp, _i32p, _vp]),
        "toep_renderer_path": (ctypes.c_int, [_vp]),
        "toep_renderer_kernels": (ctypes.c_int, [_vp, ctypes.c_int64]),
        "toep_mixer_create": (ctypes.c_int, [_vp, _i32p, _i32, _i64, ctypes.POINTER(_vp)]),
        "toep_mixer_destroy": (ctypes.c_int, [_vp]),
        "toep_mixer_z_len": (_i64, [_vp]),
        "toep_mixer_out_len": (_i64, [_vp]),
        "toep_mixer_partial": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _vp, _i64, _vp]),
        "toep_mixer_finish": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _vp]),
        "toep_mixer_path": (ctypes.c_int, [_vp]),
        "toep_mixer_kernels": (ctypes.c_int, [_vp]),
        "toep_streamer_create": (ctypes.c_int, [_vp, _i32p, _i32, _i32, ctypes.POINTER(_vp)]),
        "toep_streamer_destroy": (ctypes.c_int, [_vp]),
        "toep_streamer_reset": (ctypes.c_int, [_vp, _vp]),
        "toep_streamer_step": (ctypes.c_int, [_vp, _vp, _i64, _vp, _i64, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == TOEP_OK:
        return
    msg = load_library().toep_last_error().decode(errors="replace")
    if rc == TOEP_ERR_INVALID:
        raise DataError(msg)
    if rc == TOEP_ERR_UNSUPPORTED:
        raise DataError("unsupported: " + msg)
    raise NativeError(msg)


# ------------------------------------------------------------ torch glue ----
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


_cuda_ok = False


def require_cuda():
    """Library loaded and a CUDA device present, else NativeUnavailable."""
    global _cuda_ok
    if _cuda_ok:
        return _torch
    load_library()
    t = torch()
    if not t.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the renderer has no CPU fallback")
    _cuda_ok = True
    return t


def stream_ptr(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return int(s.cuda_stream)


def dptr(x) -> int:
    return int(x.data_ptr())


def host_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ----------------------------------------------------------- handle types ----
class Taps:
    """Device tap table (toep_taps): CSR filters of one dense length."""

    def __init__(self, rows_taps, length: int):
        L = load_library()
        counts = [int(np.asarray(i).size) for i, _ in rows_taps]
        row_ptr = np.zeros(len(rows_taps) + 1, dtype=np.int64)
        row_ptr[1:] = np.cumsum(counts)
        if rows_taps and row_ptr[-1]:
            idx = np.concatenate([np.asarray(i, dtype=np.int64).ravel() for i, _ in rows_taps])
            val = np.concatenate([np.asarray(v, dtype=np.float32).ravel() for _, v in rows_taps])
        else:
            idx = np.zeros(1, np.int64)
            val = np.zeros(1, np.float32)
        idx = np.ascontiguousarray(idx)
        val = np.ascontiguousarray(val)
        h = _vp()
        check(L.toep_taps_create(len(rows_taps), int(length), row_ptr.ctypes.data_as(_i64p),
                                 idx.ctypes.data_as(_i64p), val.ctypes.data_as(_fp), ctypes.byref(h)))
        self._h = h
        self.rows = len(rows_taps)
        self.length = int(length)
        self.counts = np.asarray(counts, dtype=np.int64)

    @property
    def handle(self):
        return self._h

    def info(self):
        r, l, m, t = _i32(), _i32(), _i32(), _i64()
        check(load_library().toep_taps_info(self._h, ctypes.byref(r), ctypes.byref(l), ctypes.byref(m),
                                            ctypes.byref(t)))
        return {"rows": r.value, "length": l.value, "max_nnz": m.value, "total_nnz": t.value}

    def conv(self, row: int, y, out, stream=None):
        check(load_library().toep_taps_conv(self._h, int(row), dptr(y), int(y.numel()), dptr(out),
                                            stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.toep_taps_destroy(h)
            self._h = None


class NativeRenderer:
    """toep_renderer: resonance taps per ear + ear-major reflection table."""

    def __init__(self, f: np.ndarray, taps: Taps, dirs: int):
        L = load_library()
        f = np.ascontiguousarray(np.atleast_2d(f), dtype=np.float32)
        h = _vp()
        check(L.toep_renderer_create(f.ctypes.data_as(_fp), f.shape[0], f.shape[1], taps.handle, int(dirs),
                                     ctypes.byref(h)))
        self._h = h
        self.taps = taps  # keep the table alive
        self.ears, self.lf = f.shape
        self.dirs = int(dirs)

    @property
    def handle(self):
        return self._h

    def out_len(self, ny: int) -> int:
        return int(load_library().toep_renderer_out_len(self._h, int(ny)))

    def min_pitch(self, ny: int) -> int:
        return int(load_library().toep_renderer_min_pitch(self._h, int(ny)))

    def pitch(self, ny: int) -> int:
        """Recommended row pitch (128-byte rows)."""
        return int(load_library().toep_renderer_pitch(self._h, int(ny)))

    def render(self, y, out, pitch: int, stream=None):
        check(load_library().toep_renderer_render(self._h, dptr(y), int(y.numel()), dptr(out), int(pitch),
                                                  stream_ptr(stream)))

    PATHS = {1: "tensor", 0: "window", 2: "banded"}

    def kernels(self, ny: int) -> int:
        """Kernel launches render() makes for a signal of ny samples."""
        return int(load_library().toep_renderer_kernels(self._h, int(ny)))

    def path(self) -> str:
        """Which stage-2 kernel render() launches: "tensor" (tcgen05 GEMM), "window" (TMEM + FFMA2), "banded"."""
        return self.PATHS[load_library().toep_renderer_path(self._h)]

    def clear_nonfinite(self, stream=None):
        check(load_library().toep_renderer_check(self._h, None, stream_ptr(stream)))

    def nonfinite(self, stream=None) -> bool:
        """Waits for the stream; True if a kernel of this renderer read an inf/NaN input since the last call."""
        flag = ctypes.c_int32(0)
        check(load_library().toep_renderer_check(self._h, ctypes.byref(flag), stream_ptr(stream)))
        return bool(flag.value)

    def reflect(self, ear: int, yf, out, pitch: int, stream=None):
        check(load_library().toep_renderer_reflect(self._h, int(ear), dptr(yf), int(yf.numel()), dptr(out),
                                                   int(pitch), stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.toep_renderer_destroy(h)
            self._h = None


class NativeMixer:
    def __init__(self, renderer: NativeRenderer, src_dir, T: int):
        L = load_library()
        sd = np.ascontiguousarray(src_dir, dtype=np.int32)
        h = _vp()
        check(L.toep_mixer_create(renderer.handle, sd.ctypes.data_as(_i32p), sd.size, int(T), ctypes.byref(h)))
        self._h = h
        self.renderer = renderer
        self.S = sd.size
        self.T = int(T)

    def z_len(self) -> int:
        return int(load_library().toep_mixer_z_len(self._h))

    def out_len(self) -> int:
        return int(load_library().toep_mixer_out_len(self._h))

    def path(self) -> str:
        return {1: "tensor", 0: "window"}[int(load_library().toep_mixer_path(self._h))]

    def kernels(self) -> int:
        return int(load_library().toep_mixer_kernels(self._h))

    def partial(self, y, y_pitch: int, s0: int, count: int, z, z_pitch: int, stream=None):
        check(load_library().toep_mixer_partial(self._h, dptr(y), int(y_pitch), int(s0), int(count), dptr(z),
                                                int(z_pitch), stream_ptr(stream)))

    def finish(self, z, z_pitch: int, out, out_pitch: int, stream=None):
        check(load_library().toep_mixer_finish(self._h, dptr(z), int(z_pitch), dptr(out), int(out_pitch),
                                               stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.toep_mixer_destroy(h)
            self._h = None


class NativeStreamer:
    def __init__(self, renderer: NativeRenderer, src_dir, block: int):
        L = load_library()
        sd = np.ascontiguousarray(src_dir, dtype=np.int32)
        h = _vp()
        check(L.toep_streamer_create(renderer.handle, sd.ctypes.data_as(_i32p), sd.size, int(block),
                                     ctypes.byref(h)))
        self._h = h
        self.renderer = renderer
        self.S = sd.size
        self.B = int(block)

    def reset(self, stream=None):
        check(load_library().toep_streamer_reset(self._h, stream_ptr(stream)))

    def step(self, block, out, stream=None):
        pitch = block.stride(0) if block.dim() == 2 else self.B
        opitch = out.stride(0) if out.dim() == 2 else self.B
        check(load_library().toep_streamer_step(self._h, dptr(block), int(pitch), dptr(out), int(opitch),
                                                stream_ptr(stream)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.toep_streamer_destroy(h)
            self._h = None


def conv_dense_dev(y, taps, out, stream=None) -> int:
    macs = _i64()
    check(load_library().toep_conv_dense(dptr(y), int(y.numel()), dptr(taps), int(taps.numel()), dptr(out),
                                         ctypes.byref(macs), stream_ptr(stream)))
    return int(macs.value)


def conv_sparse_dev(y, indices: np.ndarray, values: np.ndarray, length: int, out, stream=None) -> int:
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    val = np.ascontiguousarray(values, dtype=np.float32)
    macs = _i64()
    check(load_library().toep_conv_sparse(dptr(y), int(y.numel()), idx.ctypes.data_as(_i64p),
                                          val.ctypes.data_as(_fp), idx.size, int(length), dptr(out),
                                          ctypes.byref(macs), stream_ptr(stream)))
    return int(macs.value)


def fft_c128(x, out, inverse: bool, stream=None) -> int:
    """out = DFT of x (complex128 CUDA tensors, power-of-two length); returns the butterfly count."""
    macs = _i64()
    check(load_library().toep_fft(dptr(x), dptr(out), int(x.numel()), 1 if inverse else 0, ctypes.byref(macs),
                                  stream_ptr(stream)))
    return int(macs.value)


def fft_spectrum(taps, n: int, stream=None):
    """complex64 CUDA tensor [n]: DFT of the float32 taps zero-padded to n."""
    t = torch()
    spec = t.empty(n, device="cuda", dtype=t.complex64)
    check(load_library().toep_fft_spectrum(dptr(taps), int(taps.numel()), int(n), dptr(spec), stream_ptr(stream)))
    return spec


def fft_conv(y, spectrum, n: int, ntaps: int, out, stream=None) -> None:
    """FFT overlap-save convolution of float32 y with the taps behind ``spectrum`` into out."""
    check(load_library().toep_fft_conv(dptr(y), int(y.numel()), dptr(spectrum), int(n), int(ntaps), dptr(out),
                                       stream_ptr(stream)))
