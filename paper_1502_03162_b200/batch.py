"""Batched entry points the per-call reference seam cannot express.

* :class:`BatchRenderer` -- one source through every (ear, direction) of a
  model set in one fused launch (BASELINE configs 1-3).  Equivalent to
  ``Renderer(model_e).render(y, d)`` for all e, d (engine/__init__.py:238-260).
* :class:`MixRenderer` -- many sources, each at one direction, summed into a
  stereo (per-ear) mix with the reflection filters applied first and the
  resonance once on the mix (configs 4 offline and 5).  Equivalent to
  ``sum_s Renderer(model_e).render(y_s, dir(s))`` by the associativity the
  paper factorizes for (tests/test_acceptance.py:283-300).
* :class:`StreamRenderer` -- the same mixdown in fixed-size blocks with
  carried overlap history (config 4), one kernel launch per block.

All arrays are CUDA tensors; nothing here touches the host except the small
tap tables at construction.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DataError


def _as_models(models):
    if isinstance(models, (list, tuple)):
        ms = list(models)
    else:
        ms = [models]
    if not ms:
        raise DataError("need at least one model (one per ear)")
    D = ms[0].num_directions
    K = ms[0].reflection_length
    lf = ms[0].resonance_taps.size
    for m in ms[1:]:
        if m.num_directions != D or m.reflection_length != K or m.resonance_taps.size != lf:
            raise DataError("all ears must share directions, reflection length and resonance length")
    return ms, D, K, lf


def model_rows(models):
    """Ear-major (indices, values) pairs; dense rows drop zeros as sparse_parts does (engine/__init__.py:148-152)."""
    rows = []
    for m in models:
        for d in range(m.num_directions):
            if m.is_sparse:
                sf = m.reflections[d]
                if sf.length != m.reflection_length:
                    raise DataError("all reflection filters of a model must share one length")
                rows.append((np.asarray(sf.indices, np.int64), np.asarray(sf.values, np.float64)))
            else:
                dense = m.reflection(d)
                idx = np.flatnonzero(dense).astype(np.int64)
                rows.append((idx, dense[idx]))
    return rows


class _ModelSet:
    def __init__(self, models):
        self.models, self.dirs, self.K, self.lf = _as_models(models)
        self.ears = len(self.models)
        f = np.stack([np.asarray(m.resonance_taps, np.float64) for m in self.models])
        if not np.all(np.isfinite(f)):
            raise DataError("taps contain non-finite values")
        self.rows = model_rows(self.models)
        _lib.require_cuda()  # no host fallback: fail before building device state
        self.row_nnz = np.array([r[0].size for r in self.rows], dtype=np.int64)
        self.taps = _lib.Taps(self.rows, self.K)
        self.native = _lib.NativeRenderer(f, self.taps, self.dirs)
        self.M = self.lf + self.K - 1
        # non-finite inputs are detected inside the kernels (a device flag, no
        # extra pass) on every path except the banded fallback for K > 497
        self.fused_check = self.K <= 497


class BatchRenderer(_ModelSet):
    """y -> out[e, d, :] = (y * f_e) * g_{e,d} for every ear and direction, fused.

    ``counters`` follows Renderer.counters: the resonance stage is counted once
    per ear and call, the reflection stage per (ear, direction).
    """

    def __init__(self, models):
        super().__init__(models)
        self.counters = {"resonance_macs": 0, "reflection_macs": 0, "calls": 0}
        self.total_nnz = int(self.row_nnz.sum())
        self._checked_out = None

    def out_len(self, ny: int) -> int:
        return ny + self.M - 1

    def alloc(self, ny: int):
        """Output buffer [ears, dirs, pitch] (pitch >= out_len, 128-byte rows)."""
        t = _lib.require_cuda()
        pitch = self.native.pitch(ny)
        return t.empty((self.ears, self.dirs, pitch), device="cuda", dtype=t.float32)

    def render_all(self, y, out=None, stream=None, check_finite: bool = True):
        """Returns a [ears, dirs, out_len] float32 view (of ``out`` when given)."""
        t = _lib.require_cuda()
        if isinstance(y, t.Tensor):
            x = y if (y.is_cuda and y.dtype == t.float32 and y.is_contiguous()) else \
                y.to(device="cuda", dtype=t.float32).contiguous()
        else:
            x = t.from_numpy(np.ascontiguousarray(getattr(y, "samples", y), dtype=np.float32)).to("cuda")
        if x.ndim != 1 or x.numel() == 0:
            raise DataError("signal must be a non-empty 1-d array")
        fused_check = check_finite and self.fused_check
        if check_finite and not fused_check and not bool(t.isfinite(x).all()):
            raise DataError("signal contains non-finite samples")
        if fused_check:
            self.native.clear_nonfinite(stream)
        ny = x.numel()
        if out is None:
            out = self.alloc(ny)
        if out is not self._checked_out:  # validated once per output buffer object
            if out.dtype != t.float32 or not out.is_cuda or out.dim() != 3 or out.shape[:2] != (self.ears, self.dirs):
                raise DataError("output must be a float32 CUDA tensor of shape [ears, dirs, pitch]")
            if out.stride(2) != 1 or out.stride(1) != out.shape[2] or out.stride(0) != out.shape[1] * out.shape[2]:
                raise DataError("output must be contiguous")
            self._checked_out = out
        pitch = out.shape[2]
        if pitch < self.out_len(ny):
            raise DataError("output pitch %d < %d samples" % (pitch, self.out_len(ny)))
        self.native.render(x, out, pitch, stream)
        if fused_check and self.native.nonfinite(stream):
            raise DataError("signal contains non-finite samples")
        self.counters["resonance_macs"] += self.ears * self.lf * ny
        self.counters["reflection_macs"] += self.total_nnz * (ny + self.lf - 1)
        self.counters["calls"] += 1
        return out[:, :, : self.out_len(ny)]

    def reflect(self, yf, ear: int, out=None, stream=None):
        """Stage 2 only for one ear: rows (yf * g_{ear,d}) for all d; yf = y*f_ear on the device."""
        t = _lib.require_cuda()
        x = yf.to(device="cuda", dtype=t.float32).contiguous()
        L = x.numel() + self.K - 1
        if out is None:
            out = t.empty((self.dirs, (L + 3) // 4 * 4), device="cuda", dtype=t.float32)
        self.native.reflect(ear, x, out, out.shape[1], stream)
        self.counters["reflection_macs"] += int(self.row_nnz[ear * self.dirs:(ear + 1) * self.dirs].sum()) * x.numel()
        return out[:, :L]


class MixRenderer(_ModelSet):
    """S sources at directions src_dir -> per-ear mix  out[e] = sum_s (y_s * f_e) * g_{e,dir(s)}.

    Computed as  out[e] = f_e * z[e],  z[e] = sum_s y_s * g_{e,dir(s)}  (reflection first).
    """

    def __init__(self, models, src_dir, T: int):
        super().__init__(models)
        self.src_dir = np.ascontiguousarray(src_dir, dtype=np.int32)
        if self.src_dir.ndim != 1 or self.src_dir.size == 0:
            raise DataError("need at least one source")
        if np.any(self.src_dir < 0) or np.any(self.src_dir >= self.dirs):
            bad = int(self.src_dir[(self.src_dir < 0) | (self.src_dir >= self.dirs)][0])
            raise DataError("direction %d out of range" % bad)
        self.S = self.src_dir.size
        self.T = int(T)
        self.mixer = _lib.NativeMixer(self.native, self.src_dir, self.T)
        self.z_len = self.mixer.z_len()
        self.out_len = self.mixer.out_len()

    @property
    def path(self) -> str:
        """"tensor" (tcgen05 GEMM over direction sums + overlap-add) or "window"
        (TMEM window + FFMA2); the tensor plan built at the first partial() may
        fall back to "window" (tables beyond shared memory)."""
        return self.mixer.path()

    @property
    def kernels(self) -> int:
        """Kernel launches per partial() call."""
        return self.mixer.kernels()

    def alloc_z(self):
        t = _lib.require_cuda()
        return t.zeros((self.ears, (self.z_len + 3) // 4 * 4), device="cuda", dtype=t.float32)

    def partial(self, y, s0: int = 0, count: int | None = None, z=None, stream=None, check_finite: bool = True):
        """z[e] = sum over sources [s0, s0+count) of y_s * g_{e,dir(s)}; y row i is source s0+i.

        ``check_finite`` raises DataError (after the launch; the check is fused
        into the kernel's source reads) if any source sample is inf or NaN."""
        t = _lib.require_cuda()
        count = self.S - s0 if count is None else int(count)
        if y.dim() != 2 or y.shape[0] < count or y.shape[1] < self.T or y.stride(1) != 1:
            raise DataError("sources must be a [count, >=T] row-major CUDA tensor")
        if y.dtype != t.float32 or not y.is_cuda:
            raise DataError("sources must be float32 CUDA tensors")
        if z is None:
            z = self.alloc_z()
        if check_finite:
            self.native.clear_nonfinite(stream)
        self.mixer.partial(y, y.stride(0), s0, count, z, z.stride(0), stream)
        if check_finite and self.native.nonfinite(stream):
            raise DataError("signal contains non-finite samples")
        return z

    def finish(self, z, out=None, stream=None):
        t = _lib.require_cuda()
        if out is None:
            out = t.empty((self.ears, (self.out_len + 3) // 4 * 4), device="cuda", dtype=t.float32)
        self.mixer.finish(z, z.stride(0), out, out.stride(0), stream)
        return out[:, : self.out_len]

    def render(self, y, stream=None, check_finite: bool = True):
        return self.finish(self.partial(y, stream=stream, check_finite=check_finite), stream=stream)


class StreamRenderer(_ModelSet):
    """Block-by-block mixdown with carried history: step n returns samples
    [n*B, (n+1)*B) of :class:`MixRenderer`'s output for the concatenated input."""

    def __init__(self, models, src_dir, block: int):
        super().__init__(models)
        self.src_dir = np.ascontiguousarray(src_dir, dtype=np.int32)
        if np.any(self.src_dir < 0) or np.any(self.src_dir >= self.dirs):
            raise DataError("direction out of range")
        self.S = self.src_dir.size
        self.B = int(block)
        self.streamer = _lib.NativeStreamer(self.native, self.src_dir, self.B)

    def reset(self, stream=None):
        self.streamer.reset(stream)
        self.native.clear_nonfinite(stream)

    def nonfinite(self, stream=None) -> bool:
        """True if any block since the last reset/query held an inf or NaN sample
        (flag set inside the step kernel; this call waits for the stream)."""
        return self.native.nonfinite(stream)

    def step(self, block, out=None, stream=None):
        t = _lib.require_cuda()
        if tuple(block.shape) != (self.S, self.B) or block.dtype != t.float32 or not block.is_cuda:
            raise DataError("block must be a float32 CUDA tensor of shape [S, B]")
        if block.stride(1) != 1:
            block = block.contiguous()  # rows may be a strided window of a resident [S, T] array
        if out is None:
            out = t.empty((self.ears, self.B), device="cuda", dtype=t.float32)
        if tuple(out.shape) != (self.ears, self.B) or out.dtype != t.float32 or not out.is_cuda or out.stride(1) != 1:
            raise DataError("out must be a float32 CUDA tensor [ears, B] with unit column stride")
        self.streamer.step(block, out, stream)
        return out

    def host_step_graph(self, host_in, host_out):
        """CUDA graph of one block from host memory and back: copy the pinned
        host block [S, B] in, step, copy the stereo block [ears, B] out.  Each
        ``replay()`` advances the stream by one block (the history carries
        over); the caller refills ``host_in`` between replays and reads
        ``host_out`` after synchronizing -- a real-time loop with one host
        launch per block."""
        t = _lib.require_cuda()
        if tuple(host_in.shape) != (self.S, self.B) or tuple(host_out.shape) != (self.ears, self.B):
            raise DataError("host buffers must be [S, B] and [ears, B]")
        if host_in.is_cuda or host_out.is_cuda or not host_in.is_pinned() or not host_out.is_pinned():
            raise DataError("host buffers must be pinned host tensors")
        self._dev_in = t.empty((self.S, self.B), device="cuda", dtype=t.float32)
        self._dev_out = t.empty((self.ears, self.B), device="cuda", dtype=t.float32)
        g = t.cuda.CUDAGraph()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            with t.cuda.graph(g, stream=s):
                self._dev_in.copy_(host_in, non_blocking=True)
                self.step(self._dev_in, out=self._dev_out)
                host_out.copy_(self._dev_out, non_blocking=True)
        t.cuda.current_stream().wait_stream(s)
        return g

    def capture(self, y, out, blocks: int | None = None):
        """CUDA graph of consecutive steps over a device-resident [S, T] input.

        Block b reads y[:, b*B:(b+1)*B] and writes out[:, b*B:(b+1)*B]; replaying
        the graph streams the whole signal with one host launch (the
        per-block host launch overhead disappears; each node is one kernel).
        """
        t = _lib.require_cuda()
        n = (y.shape[1] // self.B) if blocks is None else int(blocks)
        g = t.cuda.CUDAGraph()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            with t.cuda.graph(g, stream=s):
                for b in range(n):
                    self.step(y[:, b * self.B:(b + 1) * self.B], out=out[:, b * self.B:(b + 1) * self.B])
        t.cuda.current_stream().wait_stream(s)
        return g
