/*
 * toep_b200 -- C ABI of the B200-native sparse-HRIR renderer.
 *
 * Plain C: device pointers are `float*` in the current CUDA device's memory,
 * streams are passed as `void*` (a cudaStream_t; NULL = legacy default
 * stream), every call is stream-ordered and returns a status code.  No C++
 * exception and no torch type crosses this boundary.
 *
 * Reference interfaces replaced (paths relative to the toepnmf package,
 * pkg/src/toepnmf/):
 *   engine/_kernels.pyx:11  conv_dense(double[::1] y, double[::1] taps) -> (out, macs)
 *   engine/_kernels.pyx:28  conv_sparse(double[::1] y, long long[::1] indices,
 *                                       double[::1] values, Py_ssize_t length) -> (out, macs)
 *   engine/__init__.py:104  ConvPlan(taps, mode, block_size, backend)   (tap tables)
 *   engine/__init__.py:208  Renderer(model, mode, block_size, backend)   (per-model plan)
 *   engine/__init__.py:238  Renderer.render(y, direction)
 *   sparsify.py:67          SparseFilter(indices, values, length)       (validation rules)
 * The batched / mixdown / streaming entry points have no single reference
 * function: they are compositions of Renderer.render calls.
 *
 * Arithmetic is fp32 with fp32 accumulation (the reference computes in fp64);
 * parity target: relative L2 error <= 1e-5 against the reference.
 *
 * Threading (as the reference's plans and renderers, engine/__init__.py:16-18):
 * distinct objects may be used concurrently from any thread / stream; the
 * calls on one renderer, mixer or streamer must be ordered (one stream at a
 * time) -- they own device scratch (tensor-map caches, the fill launch's side
 * stream, the mix plan and item counter, the stream history).  Mixers and
 * streamers made from one renderer report non-finite input through that
 * renderer's flag (toep_renderer_check): order them with the renderer, or
 * give each its own renderer (the Python layer does).  Read-only queries are
 * always safe.
 */
#ifndef TOEP_B200_H
#define TOEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define TOEP_OK 0
#define TOEP_ERR_INVALID 1     /* bad argument (the Python layer raises DataError) */
#define TOEP_ERR_CUDA 2        /* CUDA runtime failure                            */
#define TOEP_ERR_NOMEM 3       /* device allocation failed                        */
#define TOEP_ERR_UNSUPPORTED 4 /* shape outside the implemented envelope          */

#define TOEP_ABI_VERSION 1

/* Message for the last failing call on this host thread ("" if none). */
const char* toep_last_error(void);
int toep_abi_version(void);
/* Streaming-multiprocessor count of the current device (148 on B200). */
int toep_sm_count(int* out);

/* ---- reference plugin seam (engine/_kernels.pyx) ------------------------ */
/* out[0 .. ny+ntaps-1) = full linear convolution of y with dense taps.
 * ref: _kernels.pyx:11-25 (conv_dense).  *macs = ntaps*ny, as the reference. */
int toep_conv_dense(const float* y, int64_t ny, const float* taps, int64_t ntaps, float* out, int64_t* macs,
                    void* stream);

/* Sparse taps given as HOST arrays (indices in [0, length) in any order,
 * repeated indices adding up -- as the reference kernel accumulates them;
 * values finite); out[0 .. ny+length-1) on the device.
 * ref: _kernels.pyx:28-44 (conv_sparse).  *macs = nnz*ny. */
int toep_conv_sparse(const float* y, int64_t ny, const int64_t* indices, const float* values, int64_t nnz,
                     int64_t length, float* out, int64_t* macs, void* stream);

/* Power-of-two DFT of n complex128 values (interleaved re, im), inverse
 * scaled by 1/n.  ref: _kernels.pyx:47-77 (fft); *macs = n/2 * log2(n).
 * in may equal out. */
int toep_fft(const double* in, double* out, int64_t n, int inverse, int64_t* macs, void* stream);
/* spectrum[n] (complex64, interleaved) = DFT of taps[0..ntaps) zero-padded to n. */
int toep_fft_spectrum(const float* taps, int64_t ntaps, int64_t n, float* spectrum, void* stream);
/* FFT overlap-save: out[0 .. ny+ntaps-1) = y * taps, blocks of n samples
 * advancing by n - ntaps + 1, with spectrum from toep_fft_spectrum.
 * ref: engine/__init__.py:178-205 (_overlap_save). */
int toep_fft_conv(const float* y, int64_t ny, const float* spectrum, int64_t n, int64_t ntaps, float* out,
                  void* stream);

/* ---- tap tables (ConvPlan.sparse_parts / SparseFilter, device resident) - */
typedef struct toep_taps toep_taps;
/* rows CSR filters of common dense length `length`, HOST arrays:
 * row_ptr[rows+1], indices[row_ptr[rows]], values[row_ptr[rows]]. */
int toep_taps_create(int32_t rows, int32_t length, const int64_t* row_ptr, const int64_t* indices,
                     const float* values, toep_taps** out);
int toep_taps_destroy(toep_taps* t);
int toep_taps_info(const toep_taps* t, int32_t* rows, int32_t* length, int32_t* max_nnz, int64_t* total_nnz);
/* One row of a table against one device signal: out[0 .. ny+length-1),
 * exactly (nothing past the end is written; any alignment). */
int toep_taps_conv(const toep_taps* t, int32_t row, const float* y, int64_t ny, float* out, void* stream);

/* ---- renderer: resonance f per ear + reflection table rows ear-major ----- */
typedef struct toep_renderer toep_renderer;
/* f_host: [ears][lf] fp32; g: ears*dirs rows (row = ear*dirs + direction). */
int toep_renderer_create(const float* f_host, int32_t ears, int32_t lf, const toep_taps* g, int32_t dirs,
                         toep_renderer** out);
int toep_renderer_destroy(toep_renderer* r);
/* Output samples per row for an input of ny samples: ny + lf + length - 2. */
int64_t toep_renderer_out_len(const toep_renderer* r, int64_t ny);
/* Minimum row pitch (floats) accepted by toep_renderer_render. */
int64_t toep_renderer_min_pitch(const toep_renderer* r, int64_t ny);
/* Recommended row pitch (floats): out_len rounded up to 32 (128-byte rows,
 * whole cache lines per store); any pitch >= min_pitch with pitch % 4 == 0
 * is accepted. */
int64_t toep_renderer_pitch(const toep_renderer* r, int64_t ny);
/* Every (ear, direction): out[row*out_pitch + t] = ((y*f_ear)*g_row)[t],
 * t < out_len; samples in [out_len, min_pitch) of a row may be written
 * (with zeros).  out must be 16-byte aligned and out_pitch % 4 == 0.
 * ref: Renderer.render (engine/__init__.py:238-260) for all directions. */
int toep_renderer_render(const toep_renderer* r, const float* y, int64_t ny, float* out, int64_t out_pitch,
                         void* stream);
/* Kernel toep_renderer_render uses for this renderer:
 * TOEP_PATH_TENSOR  -- stage 2 as a split-fp16 GEMM on the tensor cores (tcgen05.mma)
 * TOEP_PATH_WINDOW  -- TMEM sliding window + FFMA2 per sparse tap
 * TOEP_PATH_BANDED  -- banded shared-memory kernel (reflection length > 497)
 * (TOEP_RENDER_MMA=0 in the environment disables the tensor path.) */
#define TOEP_PATH_TENSOR 1
#define TOEP_PATH_WINDOW 0
#define TOEP_PATH_BANDED 2
int toep_renderer_path(const toep_renderer* r);
/* Kernel launches one toep_renderer_render call makes for a signal of ny
 * samples (the tensor path adds a concurrent launch on the SMs its clusters
 * leave idle; the banded path runs one FIR per ear first). */
int toep_renderer_kernels(const toep_renderer* r, int64_t ny);
/* Fused input check (the reference's DataError "signal contains non-finite
 * samples", engine/__init__.py:162-165): every render / reflect / mixer /
 * streamer kernel made from this renderer ORs a device flag when it reads an
 * inf or NaN input sample (no extra pass over the input).  This call waits
 * for `stream`, returns the flag in *nonfinite (0/1) and clears it;
 * nonfinite == NULL only clears it (stream-ordered, no wait).
 * (Reflection lengths > 497 take the banded fallback, which is not covered.) */
int toep_renderer_check(const toep_renderer* r, int32_t* nonfinite, void* stream);
/* Stage 2 only, every direction of one ear against a precomputed y*f
 * (length nyf): the per-direction reflection convolution of Renderer.render
 * once the resonance cache is warm (engine/__init__.py:252-260).  Row d at
 * out + d*out_pitch, nyf+K-1 samples; with more than one direction the tail
 * of a row up to the next multiple of 4 samples may be written (zeros), so
 * out_pitch % 4 == 0 and out 16-byte aligned; a single direction is written
 * exactly (any alignment). */
int toep_renderer_reflect(const toep_renderer* r, int32_t ear, const float* yf, int64_t nyf, float* out,
                          int64_t out_pitch, void* stream);

/* ---- mixdown: S sources each at one direction, summed per ear ------------- */
typedef struct toep_mixer toep_mixer;
/* src_dir_host[S]: direction index of every source; T: samples per source. */
int toep_mixer_create(const toep_renderer* r, const int32_t* src_dir_host, int32_t n_src, int64_t T,
                      toep_mixer** out);
int toep_mixer_destroy(toep_mixer* m);
int64_t toep_mixer_z_len(const toep_mixer* m);   /* T + length - 1 */
int64_t toep_mixer_out_len(const toep_mixer* m); /* T + lf + length - 2 */
/* z[e][t] = sum over sources s in [s0, s0+count) of (y_s * g_{e,dir(s)})[t]
 * (reflection first; linear, so partial sums from several calls or ranks add).
 * y: source s at y + (s - s0) * y_pitch, 16-byte aligned, y_pitch % 4 == 0.
 * Writes z[e][0 .. z_len) (no accumulation into z).  A non-finite source
 * sample sets the renderer's non-finite flag (tensor path: detected on z). */
int toep_mixer_partial(toep_mixer* m, const float* y, int64_t y_pitch, int32_t s0, int32_t count, float* z,
                       int64_t z_pitch, void* stream);
/* Kernel toep_mixer_partial uses: TOEP_PATH_TENSOR (split-fp16 GEMM over
 * direction sums on the tensor cores, then an overlap-add; the default when
 * ears x round_up(length, 8) <= 208) or TOEP_PATH_WINDOW (TMEM window + FFMA2
 * per tap; TOEP_MIX_MMA=0 in the environment forces it). */
int toep_mixer_path(const toep_mixer* m);
/* Kernel launches per toep_mixer_partial call (tensor path: main pass, fixup
 * pass for tiles outside the fp16-safe range, overhang carry + z check). */
int toep_mixer_kernels(const toep_mixer* m);
/* out[e] = f_e * z[e] (length out_len). */
int toep_mixer_finish(const toep_mixer* m, const float* z, int64_t z_pitch, float* out, int64_t out_pitch,
                      void* stream);

/* ---- streaming: fixed block size, carried overlap history ---------------- */
typedef struct toep_streamer toep_streamer;
/* block: multiple of 4 in [4, 256]; ears <= 2. */
int toep_streamer_create(const toep_renderer* r, const int32_t* src_dir_host, int32_t n_src, int32_t block,
                         toep_streamer** out);
int toep_streamer_destroy(toep_streamer* s);
/* Zero all carried history (stream-ordered). */
int toep_streamer_reset(toep_streamer* s, void* stream);
/* block: S rows of `block` new samples, source s at block + s*block_pitch
 * (block_pitch >= block, multiple of 4, block 16-byte aligned; e.g. a window
 * into a resident [S][T] array);
 * out: ear e at out + e*out_pitch, `block` samples = samples
 * [n*block, (n+1)*block) of the full mixdown after the n-th call. */
int toep_streamer_step(toep_streamer* s, const float* block, int64_t block_pitch, float* out, int64_t out_pitch,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOEP_B200_H */
