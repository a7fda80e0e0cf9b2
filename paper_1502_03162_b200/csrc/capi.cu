// C ABI implementation (include/toep_b200.h).  Validation mirrors the
// reference's DataError rules; kernels live in render_mma.cu, render.cu, fir_mix.cu and fft.cu.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include <cuda_fp16.h>

#include "../../include/toep_b200.h"
#include "launch.h"

using namespace toep;

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? TOEP_ERR_NOMEM : TOEP_ERR_CUDA, "%s: %s", where,
              cudaGetErrorString(e));
}
#define TOEP_CUDA(call)                                     \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);     \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count_cached() {
  static thread_local int dev = -1, count = 0;
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return 148;
  if (d != dev) {
    dev = d;
    if (cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, d) != cudaSuccess) count = 148;
  }
  return count;
}

inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Stream-ordered allocations come from a per-device pool that keeps freed
// memory (release threshold = max): the default pool hands memory back to the
// driver at every synchronisation, so a per-call scratch buffer after a host
// sync paid a fresh mapping (~10 ms measured on the numpy Renderer.render path).
cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      pools[dev] = nullptr;
      return nullptr;
    }
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return pools[dev];
}

template <class T>
cudaError_t pool_alloc(T** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool = scratch_pool();
  if (!pool) return cudaMallocAsync(reinterpret_cast<void**>(p), bytes, st);
  return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, st);
}

}  // namespace

// ------------------------------------------------------------ tap tables ----
struct toep_taps {
  int rows = 0, length = 0, max_nnz = 0, kwin = -1, tap_stride = 1, uniform = 0;
  long long total = 0;
  int2* d_kw = nullptr;   // col = kwin - offset (TMEM kernels)
  int2* d_raw = nullptr;  // col = offset (generic / streaming kernels)
  int* d_nnz = nullptr;
  bool stream_owned = false;  // freed with cudaFreeAsync on `owner`
  cudaStream_t owner = nullptr;
  // per-row pair tables {col, v, kwin, 0} + {nnz, 0, 0, 0} for single-row
  // convolutions on the window kernel (toep_taps_conv); one allocation
  int4* d_rowpairs = nullptr;  // [rows][tap_stride]
  int4* d_rowpnnz = nullptr;   // [rows]
};

static bool uniform_supported(int n) { return n == 4 || n == 8 || n == 12 || n == 16 || n == 24 || n == 32; }

static int taps_build(int32_t rows, int32_t length, const int64_t* row_ptr, const int64_t* indices,
                      const float* values, bool stream_owned, cudaStream_t st, toep_taps** out) {
  if (!out) return fail(TOEP_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (rows < 1) return fail(TOEP_ERR_INVALID, "need at least one filter row, got %d", rows);
  if (length < 1) return fail(TOEP_ERR_INVALID, "filter length must be at least 1");  // sparsify.py:87-88
  if (!row_ptr) return fail(TOEP_ERR_INVALID, "null row_ptr");
  if (row_ptr[0] != 0) return fail(TOEP_ERR_INVALID, "row_ptr[0] must be 0");
  int max_nnz = 0;
  bool uni = true;
  for (int r = 0; r < rows; ++r) {
    const long long a = row_ptr[r], b = row_ptr[r + 1];
    if (b < a) return fail(TOEP_ERR_INVALID, "row_ptr must be non-decreasing (row %d)", r);
    const long long n = b - a;
    if (n > length) return fail(TOEP_ERR_INVALID, "row %d has %lld taps for length %d", r, n, length);
    for (long long k = a; k < b; ++k) {
      const long long o = indices[k];
      if (o < 0 || o >= length)  // sparsify.py:83-84
        return fail(TOEP_ERR_INVALID, "indices must lie in [0, %d) (row %d)", length, r);
      if (k > a && o <= indices[k - 1])  // sparsify.py:81-82
        return fail(TOEP_ERR_INVALID, "indices must be strictly increasing (row %d)", r);
      if (!std::isfinite(values[k])) return fail(TOEP_ERR_INVALID, "values must be finite (row %d)", r);
    }
    if (r > 0 && n != max_nnz) uni = false;
    max_nnz = std::max<int>(max_nnz, (int)n);
  }
  auto* t = new (std::nothrow) toep_taps();
  if (!t) return fail(TOEP_ERR_NOMEM, "host allocation failed");
  t->rows = rows;
  t->length = length;
  t->max_nnz = max_nnz;
  t->total = row_ptr[rows];
  t->kwin = render_kwin_for(length);
  t->tap_stride = std::max(2, (max_nnz + 1) & ~1);  // even: tap rows are whole 16-byte units (bulk copies)
  t->uniform = (uni && uniform_supported(max_nnz)) ? 1 : 0;
  t->stream_owned = stream_owned;
  t->owner = st;
  const size_t n = (size_t)rows * t->tap_stride;
  std::vector<int2> kw(n), raw(n);
  std::vector<int> nnz(rows);
  for (int r = 0; r < rows; ++r) {
    const long long a = row_ptr[r], b = row_ptr[r + 1];
    nnz[r] = (int)(b - a);
    for (int k = 0; k < t->tap_stride; ++k) {
      int o = 0;
      float v = 0.f;
      if (a + k < b) {
        o = (int)indices[a + k];
        v = values[a + k];
      }
      int vb;
      memcpy(&vb, &v, 4);
      raw[(size_t)r * t->tap_stride + k] = make_int2(o, vb);
      kw[(size_t)r * t->tap_stride + k] = make_int2(t->kwin > 0 ? t->kwin - o : 0, vb);
    }
  }
  std::vector<int4> rp;  // row paired with an empty row: {colA, vA, kwin, 0}, then per-row {nnz, 0, 0, 0}
  if (t->kwin > 0) {
    rp.resize(n + rows);
    for (size_t i = 0; i < n; ++i) rp[i] = make_int4(kw[i].x, kw[i].y, t->kwin, 0);
    for (int r = 0; r < rows; ++r) rp[n + r] = make_int4(nnz[r], 0, 0, 0);
  }
  cudaError_t e;
  if (stream_owned) {
    e = pool_alloc(&t->d_kw, n * sizeof(int2), st);
    if (e == cudaSuccess) e = pool_alloc(&t->d_raw, n * sizeof(int2), st);
    if (e == cudaSuccess) e = pool_alloc(&t->d_nnz, rows * sizeof(int), st);
    if (e == cudaSuccess && !rp.empty()) e = pool_alloc(&t->d_rowpairs, rp.size() * sizeof(int4), st);
  } else {
    e = cudaMalloc(&t->d_kw, n * sizeof(int2));
    if (e == cudaSuccess) e = cudaMalloc(&t->d_raw, n * sizeof(int2));
    if (e == cudaSuccess) e = cudaMalloc(&t->d_nnz, rows * sizeof(int));
    if (e == cudaSuccess && !rp.empty()) e = cudaMalloc(&t->d_rowpairs, rp.size() * sizeof(int4));
  }
  if (t->d_rowpairs) t->d_rowpnnz = t->d_rowpairs + n;
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->d_kw, kw.data(), n * sizeof(int2), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->d_raw, raw.data(), n * sizeof(int2), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->d_nnz, nnz.data(), rows * sizeof(int), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !rp.empty())
    e = cudaMemcpyAsync(t->d_rowpairs, rp.data(), rp.size() * sizeof(int4), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !stream_owned) e = cudaStreamSynchronize(st);  // host staging vectors die here
  if (e != cudaSuccess) {
    toep_taps_destroy(t);
    return cuda_fail(e, "toep_taps_create");
  }
  *out = t;
  return TOEP_OK;
}

extern "C" {

const char* toep_last_error(void) { return g_err; }
int toep_abi_version(void) { return TOEP_ABI_VERSION; }
int toep_sm_count(int* out) {
  if (!out) return fail(TOEP_ERR_INVALID, "null output");
  int d = 0;
  TOEP_CUDA(cudaGetDevice(&d));
  TOEP_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, d));
  return TOEP_OK;
}

int toep_taps_create(int32_t rows, int32_t length, const int64_t* row_ptr, const int64_t* indices,
                     const float* values, toep_taps** out) {
  return taps_build(rows, length, row_ptr, indices, values, false, nullptr, out);
}

int toep_taps_destroy(toep_taps* t) {
  if (!t) return TOEP_OK;
  if (t->stream_owned) {
    if (t->d_kw) cudaFreeAsync(t->d_kw, t->owner);
    if (t->d_raw) cudaFreeAsync(t->d_raw, t->owner);
    if (t->d_nnz) cudaFreeAsync(t->d_nnz, t->owner);
    if (t->d_rowpairs) cudaFreeAsync(t->d_rowpairs, t->owner);
  } else {
    if (t->d_kw) cudaFree(t->d_kw);
    if (t->d_raw) cudaFree(t->d_raw);
    if (t->d_nnz) cudaFree(t->d_nnz);
    if (t->d_rowpairs) cudaFree(t->d_rowpairs);  // d_rowpnnz lives in the same allocation
  }
  delete t;
  return TOEP_OK;
}

int toep_taps_info(const toep_taps* t, int32_t* rows, int32_t* length, int32_t* max_nnz, int64_t* total_nnz) {
  if (!t) return fail(TOEP_ERR_INVALID, "null table");
  if (rows) *rows = t->rows;
  if (length) *length = t->length;
  if (max_nnz) *max_nnz = t->max_nnz;
  if (total_nnz) *total_nnz = t->total;
  return TOEP_OK;
}

}  // extern "C"

// Stage-2 ("reflection") launch over `nrows` consecutive rows of a table,
// all reading the same input signal x (nx samples).  `pairs`/`pnnz` are the
// rows' pair-interleaved taps (k_pair_taps); null -> built here for this call.
static int reflect_rows(const toep_taps* t, int row0, int nrows, const int4* pairs, const int4* pnnz, const float* x,
                        long long nx, float* out, long long out_pitch, cudaStream_t st, int* nonfinite = nullptr,
                        bool padded_out = false) {
  const long long out_len = nx + t->length - 1;
  if (nrows == 1 && !nonfinite && nx <= (1LL << 20)) {
    // one row of a per-call convolution: the banded kernel is one launch with
    // exact-length writes (the TMEM-window kernel's persistent grid, TMEM
    // allocation and 16-byte tail handling cost more than its speed wins at this size)
    SparseGenericArgs g{};
    g.x = x;
    g.nx = nx;
    g.x_pitch = 0;
    g.rows_per_x = 1;
    g.taps = t->d_raw + (size_t)row0 * t->tap_stride;
    g.row_nnz = t->d_nnz + row0;
    g.tap_stride = t->tap_stride;
    g.rows = 1;
    g.out = out;
    g.out_len = out_len;
    g.out_pitch = out_len;
    cudaError_t e = launch_sparse_generic(g, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_sparse_generic");
    return TOEP_OK;
  }
  if (t->kwin > 0 && nrows == 1 && !padded_out && (out_len % 4 != 0 || !aligned16(out))) {
    // one row, exactly out_len samples: the kernel's stores move whole 16-byte
    // units, so it renders into a padded scratch row that is copied out exact
    float* row = nullptr;
    TOEP_CUDA(pool_alloc(&row, (size_t)round_up(out_len, 4) * sizeof(float), st));
    int rc = reflect_rows(t, row0, 1, pairs, pnnz, x, nx, row, 0, st, nonfinite, true);
    if (rc == TOEP_OK) {
      cudaError_t e = cudaMemcpyAsync(out, row, (size_t)out_len * sizeof(float), cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) rc = cuda_fail(e, "copy of the rendered row");
    }
    cudaFreeAsync(row, st);
    return rc;
  }
  if (t->kwin > 0) {
    if (!aligned16(out) || (nrows > 1 && out_pitch % 4 != 0))
      return fail(TOEP_ERR_INVALID, "output must be 16-byte aligned with a pitch multiple of 4");
    const int P = (nrows + 1) / 2;
    int4* tmp = nullptr;
    if (!pairs) {
      TOEP_CUDA(pool_alloc(&tmp, (size_t)P * (t->tap_stride + 1) * sizeof(int4), st));
      cudaError_t ep = launch_pair_taps(t->d_kw + (size_t)row0 * t->tap_stride, t->d_nnz + row0, 1, nrows,
                                        t->tap_stride, t->kwin, tmp, tmp + (size_t)P * t->tap_stride, st);
      if (ep != cudaSuccess) {
        cudaFreeAsync(tmp, st);
        return cuda_fail(ep, "launch_pair_taps");
      }
      pairs = tmp;
      pnnz = tmp + (size_t)P * t->tap_stride;
    }
    RenderArgs a{};
    a.x = x;
    a.nx = nx;
    a.x_pitch = 0;
    a.f = nullptr;
    a.lf_pad = 0;
    a.pairs = pairs;
    a.pair_nnz = pnnz;
    a.pairs_per_ear = P;
    a.tap_stride = t->tap_stride;
    a.uniform_nnz = t->uniform;
    a.tap_stride_nnz = t->max_nnz;
    a.dirs = nrows;
    a.ears = 1;
    a.n_tiles = (int)((out_len + kW - 1) / kW);
    a.n_items = (long long)nrows * a.n_tiles;  // work units (direction x tile)
    a.out = out;
    a.out_pitch = out_pitch;
    a.out_len = out_len;
    a.nonfinite = nonfinite;
    RenderMaps maps;
    cudaError_t e = make_render_maps(out, nrows, out_len, out_pitch, &maps);
    if (e == cudaSuccess) e = launch_render(a, maps, t->kwin, false, sm_count_cached(), st);
    if (tmp) cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_render(stage 2)");
    return TOEP_OK;
  }
  SparseGenericArgs g{};
  g.x = x;
  g.nx = nx;
  g.x_pitch = 0;
  g.rows_per_x = 1;
  g.taps = t->d_raw + (size_t)row0 * t->tap_stride;
  g.row_nnz = t->d_nnz + row0;
  g.tap_stride = t->tap_stride;
  g.rows = nrows;
  g.out = out;
  g.out_len = out_len;
  g.out_pitch = out_pitch;
  cudaError_t e = launch_sparse_generic(g, st);
  if (e != cudaSuccess) return cuda_fail(e, "launch_sparse_generic");
  return TOEP_OK;
}

static int dense_fir(const float* x, long long nx, long long x_pitch, const float* h_pad, int nh_pad, int h_pitch,
                     int channels, float* out, long long out_len, long long out_pitch, cudaStream_t st,
                     int nh = -1) {
  FirArgs a{};
  a.x = x;
  a.nx = nx;
  a.x_pitch = x_pitch;
  a.h = h_pad;
  a.nh_pad = nh_pad;
  a.nh = nh < 0 ? nh_pad : nh;
  a.h_pitch = h_pitch;
  a.out = out;
  a.out_len = out_len;
  a.out_pitch = out_pitch;
  a.channels = channels;
  cudaError_t e = launch_fir(a, st);
  if (e != cudaSuccess) return cuda_fail(e, "launch_fir");
  return TOEP_OK;
}

extern "C" {

int toep_taps_conv(const toep_taps* t, int32_t row, const float* y, int64_t ny, float* out, void* stream) {
  if (!t) return fail(TOEP_ERR_INVALID, "null table");
  if (row < 0 || row >= t->rows) return fail(TOEP_ERR_INVALID, "row %d out of range", row);
  if (ny < 1 || !y || !out) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  cudaStream_t st = S(stream);
  if (t->kwin > 0)
    return reflect_rows(t, row, 1, t->d_rowpairs + (size_t)row * t->tap_stride, t->d_rowpnnz + row, y, ny, out, 0,
                        st);
  return reflect_rows(t, row, 1, nullptr, nullptr, y, ny, out, 0, st);
}

int toep_conv_dense(const float* y, int64_t ny, const float* taps, int64_t ntaps, float* out, int64_t* macs,
                    void* stream) {
  if (ny < 1 || !y) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (ntaps < 1 || !taps) return fail(TOEP_ERR_INVALID, "taps must be a non-empty 1-d array");
  if (!out) return fail(TOEP_ERR_INVALID, "null output");
  cudaStream_t st = S(stream);
  const long long nh_pad = round_up(ntaps, 16);
  if (nh_pad > (1LL << 30)) return fail(TOEP_ERR_UNSUPPORTED, "too many taps");
  // one launch: the FIR kernel reads taps past ntaps as zeros
  const int rc = dense_fir(y, ny, 0, taps, (int)nh_pad, 0, 1, out, ny + ntaps - 1, 0, st, (int)ntaps);
  if (rc == TOEP_OK && macs) *macs = (int64_t)ntaps * ny;  // _kernels.pyx:24
  return rc;
}

int toep_conv_sparse(const float* y, int64_t ny, const int64_t* indices, const float* values, int64_t nnz,
                     int64_t length, float* out, int64_t* macs, void* stream) {
  if (ny < 1 || !y) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (length < 1 || length > (1LL << 30)) return fail(TOEP_ERR_INVALID, "bad filter length");
  if (nnz < 0 || (nnz > 0 && (!indices || !values))) return fail(TOEP_ERR_INVALID, "bad tap arrays");
  cudaStream_t st = S(stream);
  // the reference kernel takes the taps in any order, repeated offsets adding
  // up (_kernels.pyx:38-43): sort by offset and merge repeats (in double)
  // into the strictly increasing form the tap tables hold
  std::vector<int64_t> ci;
  std::vector<float> cv;
  {
    std::vector<int64_t> ord(nnz);
    for (int64_t k = 0; k < nnz; ++k) {
      if (indices[k] < 0 || indices[k] >= length)
        return fail(TOEP_ERR_INVALID, "indices must lie in [0, %lld)", (long long)length);
      if (!std::isfinite(values[k])) return fail(TOEP_ERR_INVALID, "values must be finite");
      ord[k] = k;
    }
    std::stable_sort(ord.begin(), ord.end(), [indices](int64_t x, int64_t y2) { return indices[x] < indices[y2]; });
    for (int64_t k = 0; k < nnz;) {
      double acc = 0.0;
      int64_t q = k;
      while (q < nnz && indices[ord[q]] == indices[ord[k]]) acc += values[ord[q++]];
      ci.push_back(indices[ord[k]]);
      cv.push_back((float)acc);
      k = q;
    }
  }
  const int64_t row_ptr[2] = {0, (int64_t)ci.size()};
  toep_taps* t = nullptr;
  int rc = taps_build(1, (int32_t)length, row_ptr, ci.data(), cv.data(), true, st, &t);
  if (rc != TOEP_OK) return rc;
  rc = reflect_rows(t, 0, 1, t->d_rowpairs, t->d_rowpnnz, y, ny, out, 0, st);
  toep_taps_destroy(t);
  if (rc == TOEP_OK && macs) *macs = nnz * ny;  // _kernels.pyx:43
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------------ FFT ----
static bool pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

extern "C" {

int toep_fft(const double* in, double* out, int64_t n, int inverse, int64_t* macs, void* stream) {
  if (!pow2(n)) return fail(TOEP_ERR_INVALID, "transform length must be a power of two, got %lld", (long long)n);
  if (!in || !out) return fail(TOEP_ERR_INVALID, "null buffer");
  cudaStream_t st = S(stream);
  int logn = 0;
  while ((1LL << logn) < n) ++logn;
  if (macs) *macs = n > 1 ? (n / 2) * logn : 0;  // butterflies, _kernels.pyx:72
  double* dst = out;
  double* tmp = nullptr;
  if (in == out && fft_needs_distinct(n, true)) {
    TOEP_CUDA(pool_alloc(&tmp, (size_t)n * 2 * sizeof(double), st));
    dst = tmp;
  }
  cudaError_t e = launch_fft_c128(in, dst, n, inverse != 0, st);
  if (e == cudaSuccess && tmp) e = cudaMemcpyAsync(out, tmp, (size_t)n * 2 * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (tmp) cudaFreeAsync(tmp, st);
  return e == cudaSuccess ? TOEP_OK : cuda_fail(e, "toep_fft");
}

int toep_fft_spectrum(const float* taps, int64_t ntaps, int64_t n, float* spectrum, void* stream) {
  if (!pow2(n)) return fail(TOEP_ERR_INVALID, "transform length must be a power of two, got %lld", (long long)n);
  if (ntaps < 1 || ntaps > n || !taps || !spectrum) return fail(TOEP_ERR_INVALID, "bad taps for a %lld-point spectrum", (long long)n);
  cudaStream_t st = S(stream);
  float* tmp = nullptr;
  TOEP_CUDA(pool_alloc(&tmp, (size_t)n * 2 * sizeof(float), st));
  cudaError_t e = launch_fft_spectrum(taps, ntaps, n, spectrum, tmp, st);
  cudaFreeAsync(tmp, st);
  return e == cudaSuccess ? TOEP_OK : cuda_fail(e, "toep_fft_spectrum");
}

int toep_fft_conv(const float* y, int64_t ny, const float* spectrum, int64_t n, int64_t ntaps, float* out,
                  void* stream) {
  if (ny < 1 || !y) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (!pow2(n) || n < 2) return fail(TOEP_ERR_INVALID, "block size must be a power of two >= 2, got %lld", (long long)n);
  if (ntaps < 1 || ntaps > n) return fail(TOEP_ERR_INVALID, "block size %lld is smaller than the %lld-tap filter", (long long)n, (long long)ntaps);
  if (!spectrum || !out) return fail(TOEP_ERR_INVALID, "null buffer");
  cudaStream_t st = S(stream);
  const long long sb = fft_conv_scratch_bytes(ny, n, ntaps);
  float* scratch = nullptr;
  if (sb > 0) TOEP_CUDA(pool_alloc(&scratch, (size_t)sb, st));
  cudaError_t e = launch_fft_conv(y, ny, spectrum, n, ntaps, out, scratch, st);
  if (scratch) cudaFreeAsync(scratch, st);
  return e == cudaSuccess ? TOEP_OK : cuda_fail(e, "toep_fft_conv");
}

}  // extern "C"

// -------------------------------------------------------------- renderer ----
struct toep_renderer {
  int ears = 0, lf = 0, lf_pad = 0, dirs = 0, pairs_per_ear = 0;
  const toep_taps* g = nullptr;
  float* d_f = nullptr;      // [ears][lf_pad]
  int4* d_pairs = nullptr;   // [ears][pairs_per_ear][tap_stride] pair-interleaved taps (k_render)
  int4* d_pnnz = nullptr;    // [ears][pairs_per_ear]
  int* d_nonfinite = nullptr;  // sticky flag: a kernel read a non-finite input sample
  int4* d_epairs = nullptr;    // [dirs][tap_stride] ear-interleaved taps (mixdown)
  void* d_gmma = nullptr;      // tensor-core operand tables (render_mma.cu), null if unsupported
  int* d_gexp = nullptr;       // [ears][chunks][129] G row exponents + wide flag
  MmaFillStreams fill;         // this renderer's side stream for the concurrent fill launch
  // last output tensor map (encoding costs microseconds of host time per call)
  std::mutex map_mu;
  const float* map_out = nullptr;
  long long map_pitch = -1, map_len = -1;
  CUtensorMap map{};
};

// TOEP_RENDER_MMA=0 selects the FFMA/TMEM-window kernel for every render (A/B runs)
static bool render_mma_enabled() {
  const char* ev = getenv("TOEP_RENDER_MMA");
  return !(ev && atoi(ev) == 0);
}

extern "C" {

int toep_renderer_create(const float* f_host, int32_t ears, int32_t lf, const toep_taps* g, int32_t dirs,
                         toep_renderer** out) {
  if (!out) return fail(TOEP_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (ears < 1) return fail(TOEP_ERR_INVALID, "need at least one ear");
  if (lf < 1 || !f_host) return fail(TOEP_ERR_INVALID, "resonance taps must be a non-empty 1-d array");
  if (!g) return fail(TOEP_ERR_INVALID, "null reflection table");
  if (dirs < 1 || (long long)dirs * ears != g->rows)
    return fail(TOEP_ERR_INVALID, "table has %d rows, expected ears*dirs = %lld", g->rows, (long long)dirs * ears);
  for (long long i = 0; i < (long long)ears * lf; ++i)
    if (!std::isfinite(f_host[i])) return fail(TOEP_ERR_INVALID, "taps contain non-finite values");
  auto* r = new (std::nothrow) toep_renderer();
  if (!r) return fail(TOEP_ERR_NOMEM, "host allocation failed");
  r->ears = ears;
  r->lf = lf;
  r->lf_pad = (int)round_up(lf, 16);
  r->dirs = dirs;
  r->g = g;
  std::vector<float> fp((size_t)ears * r->lf_pad, 0.f);
  for (int e = 0; e < ears; ++e)
    for (int j = 0; j < lf; ++j) fp[(size_t)e * r->lf_pad + j] = f_host[(size_t)e * lf + j];
  cudaError_t e = cudaMalloc(&r->d_f, fp.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&r->d_nonfinite, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(r->d_nonfinite, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(r->d_f, fp.data(), fp.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (g->kwin > 0) {
    r->pairs_per_ear = (dirs + 1) / 2;
    const size_t np = (size_t)ears * r->pairs_per_ear;
    if (e == cudaSuccess) e = cudaMalloc(&r->d_pairs, np * g->tap_stride * sizeof(int4));
    if (e == cudaSuccess) e = cudaMalloc(&r->d_pnnz, np * sizeof(int4));
    if (e == cudaSuccess)
      e = launch_pair_taps(g->d_kw, g->d_nnz, ears, dirs, g->tap_stride, g->kwin, r->d_pairs, r->d_pnnz, nullptr);
    if (e == cudaSuccess && ears <= 2) e = cudaMalloc(&r->d_epairs, (size_t)dirs * g->tap_stride * sizeof(int4));
    if (e == cudaSuccess && ears <= 2)
      e = launch_ear_pair_taps(g->d_kw, dirs, ears, g->tap_stride, g->kwin, r->d_epairs, nullptr);
    if (e == cudaSuccess && render_mma_supported(g->length, r->lf_pad)) {
      const int cn = render_mma_chunk(), nch = (dirs + cn - 1) / cn;
      e = cudaMalloc(&r->d_gmma, render_mma_gbytes(ears, dirs, g->length));
      (void)nch;
      if (e == cudaSuccess) e = cudaMalloc(&r->d_gexp, render_mma_gexp_ints(ears, dirs) * sizeof(int));
      if (e == cudaSuccess)
        e = build_render_mma_tables(g->d_raw, g->d_nnz, dirs, ears, g->tap_stride, g->length, r->d_gmma,
                                    r->d_gexp, nullptr);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r->fill.side, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->fill.fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r->fill.join, cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    toep_renderer_destroy(r);
    return cuda_fail(e, "toep_renderer_create");
  }
  *out = r;
  return TOEP_OK;
}

int toep_renderer_destroy(toep_renderer* r) {
  if (!r) return TOEP_OK;
  if (r->d_f) cudaFree(r->d_f);
  if (r->d_nonfinite) cudaFree(r->d_nonfinite);
  if (r->d_epairs) cudaFree(r->d_epairs);
  if (r->d_gmma) cudaFree(r->d_gmma);
  if (r->d_gexp) cudaFree(r->d_gexp);
  if (r->fill.side) cudaStreamDestroy(r->fill.side);
  if (r->fill.fork) cudaEventDestroy(r->fill.fork);
  if (r->fill.join) cudaEventDestroy(r->fill.join);
  if (r->d_pairs) cudaFree(r->d_pairs);
  if (r->d_pnnz) cudaFree(r->d_pnnz);
  delete r;
  return TOEP_OK;
}

int64_t toep_renderer_out_len(const toep_renderer* r, int64_t ny) {
  return r ? ny + r->lf + r->g->length - 2 : -1;
}
int64_t toep_renderer_min_pitch(const toep_renderer* r, int64_t ny) {
  return r ? round_up(toep_renderer_out_len(r, ny), 4) : -1;
}

// rows on 128-byte boundaries: every TMA store box row then covers whole
// cache lines (the tensor path's store stream is ~1.3x faster than at a
// 16-byte-aligned pitch; tools/microbench/tma_store_rate.cu)
int64_t toep_renderer_pitch(const toep_renderer* r, int64_t ny) {
  return r ? round_up(toep_renderer_out_len(r, ny), 32) : -1;
}

// tensor-core path unless the taps are so sparse (<= 8 per row) that the FFMA
// kernel already meets the write roofline while the GEMM pays for KPAD > 128
// zero columns (cfg3 sweep)
static int renderer_path(const toep_renderer* r) {
  const toep_taps* g = r->g;
  if (r->d_gmma && render_mma_enabled() && !(g->max_nnz <= 8 && render_mma_kpad(g->length) > 128))
    return TOEP_PATH_TENSOR;
  return g->kwin > 0 ? TOEP_PATH_WINDOW : TOEP_PATH_BANDED;
}

int toep_renderer_path(const toep_renderer* r) { return r ? renderer_path(r) : -1; }

int toep_renderer_kernels(const toep_renderer* r, int64_t ny) {
  if (!r || ny < 1) return -1;
  switch (renderer_path(r)) {
    case TOEP_PATH_TENSOR:
      return render_mma_launches((int)((toep_renderer_out_len(r, ny) + 127) / 128), render_mma_kpad(r->g->length),
                                 r->lf_pad, sm_count_cached());
    case TOEP_PATH_WINDOW:
      return 1;
    default:
      return r->ears + 1;  // k_fir per ear, then k_sparse_generic
  }
}

int toep_renderer_check(const toep_renderer* r, int32_t* nonfinite, void* stream) {
  if (!r) return fail(TOEP_ERR_INVALID, "null renderer");
  cudaStream_t st = S(stream);
  if (!nonfinite) {  // clear only (stream-ordered, no wait)
    TOEP_CUDA(cudaMemsetAsync(r->d_nonfinite, 0, sizeof(int), st));
    return TOEP_OK;
  }
  int h = 0;
  TOEP_CUDA(cudaMemcpyAsync(&h, r->d_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
  TOEP_CUDA(cudaMemsetAsync(r->d_nonfinite, 0, sizeof(int), st));
  TOEP_CUDA(cudaStreamSynchronize(st));
  *nonfinite = h;
  return TOEP_OK;
}

int toep_renderer_render(const toep_renderer* r, const float* y, int64_t ny, float* out, int64_t out_pitch,
                         void* stream) {
  if (!r) return fail(TOEP_ERR_INVALID, "null renderer");
  if (ny < 1 || !y) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (!out) return fail(TOEP_ERR_INVALID, "null output");
  const long long out_len = toep_renderer_out_len(r, ny);
  const long long rows = (long long)r->ears * r->dirs;
  if (rows > 1 && out_pitch < out_len) return fail(TOEP_ERR_INVALID, "output pitch %lld < %lld", (long long)out_pitch, out_len);
  cudaStream_t st = S(stream);
  const toep_taps* g = r->g;
  if (renderer_path(r) == TOEP_PATH_TENSOR) {
    if (!aligned16(out) || (rows > 1 && out_pitch % 4 != 0))
      return fail(TOEP_ERR_INVALID, "output must be 16-byte aligned with a pitch multiple of 4");
    RenderMmaArgs a{};
    a.x = y;
    a.nx = ny;
    a.f = r->d_f;
    a.lf_pad = r->lf_pad;
    a.g = r->d_gmma;
    a.gexp = r->d_gexp;
    a.kpad = render_mma_kpad(g->length);
    a.nchunks = (r->dirs + render_mma_chunk() - 1) / render_mma_chunk();
    a.dirs = r->dirs;
    a.ears = r->ears;
    a.n_titems = (int)((out_len + 127) / 128);
    a.out = out;
    a.out_pitch = out_pitch;
    a.out_len = out_len;
    a.nonfinite = r->d_nonfinite;
    CUtensorMap map;
    {
      auto* rm = const_cast<toep_renderer*>(r);
      const long long pitch = rows > 1 ? out_pitch : round_up(out_len, 4);
      std::lock_guard<std::mutex> lk(rm->map_mu);
      if (rm->map_out != out || rm->map_pitch != pitch || rm->map_len != out_len) {
        cudaError_t em = make_render_mma_map(out, r->ears, r->dirs, out_len, pitch, &rm->map);
        if (em != cudaSuccess) {
          rm->map_out = nullptr;
          return cuda_fail(em, "tensor map (output rows)");
        }
        rm->map_out = out;
        rm->map_pitch = pitch;
        rm->map_len = out_len;
      }
      map = rm->map;
    }
    cudaError_t e = launch_render_mma(a, map, r->fill, sm_count_cached(), st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_render_mma");
    return TOEP_OK;
  }
  if (g->kwin > 0) {
    if (!aligned16(out) || (rows > 1 && out_pitch % 4 != 0))
      return fail(TOEP_ERR_INVALID, "output must be 16-byte aligned with a pitch multiple of 4");
    RenderArgs a{};
    a.x = y;
    a.nx = ny;
    a.f = r->d_f;
    a.lf_pad = r->lf_pad;
    a.pairs = r->d_pairs;
    a.pair_nnz = r->d_pnnz;
    a.pairs_per_ear = r->pairs_per_ear;
    a.tap_stride = g->tap_stride;
    a.uniform_nnz = g->uniform;
    a.tap_stride_nnz = g->max_nnz;
    a.dirs = r->dirs;
    a.ears = r->ears;
    a.n_tiles = (int)((out_len + kW - 1) / kW);
    a.n_items = (long long)a.ears * a.dirs * a.n_tiles;  // work units (direction x tile)
    a.out = out;
    a.out_pitch = out_pitch;
    a.out_len = out_len;
    a.nonfinite = r->d_nonfinite;
    RenderMaps maps;
    cudaError_t e = make_render_maps(out, rows, out_len, out_pitch, &maps);
    if (e != cudaSuccess) return cuda_fail(e, "tensor map (output rows)");
    e = launch_render(a, maps, g->kwin, true, sm_count_cached(), st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_render");
    return TOEP_OK;
  }
  // long reflection filters: y*f per ear into scratch, then the banded kernel
  const long long nyf = ny + r->lf - 1;
  const long long pitch = round_up(nyf, 4);
  float* yf = nullptr;
  TOEP_CUDA(pool_alloc(&yf, (size_t)pitch * r->ears * sizeof(float), st));
  int rc = TOEP_OK;
  for (int e = 0; e < r->ears && rc == TOEP_OK; ++e)
    rc = dense_fir(y, ny, 0, r->d_f + (size_t)e * r->lf_pad, r->lf_pad, 0, 1, yf + e * pitch, nyf, 0, st);
  if (rc == TOEP_OK) {
    SparseGenericArgs ga{};
    ga.x = yf;
    ga.nx = nyf;
    ga.x_pitch = pitch;
    ga.rows_per_x = r->dirs;
    ga.taps = g->d_raw;
    ga.row_nnz = g->d_nnz;
    ga.tap_stride = g->tap_stride;
    ga.rows = (int)rows;
    ga.out = out;
    ga.out_len = out_len;
    ga.out_pitch = out_pitch;
    cudaError_t e = launch_sparse_generic(ga, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "launch_sparse_generic");
  }
  cudaFreeAsync(yf, st);
  return rc;
}

int toep_renderer_reflect(const toep_renderer* r, int32_t ear, const float* yf, int64_t nyf, float* out,
                          int64_t out_pitch, void* stream) {
  if (!r) return fail(TOEP_ERR_INVALID, "null renderer");
  if (ear < 0 || ear >= r->ears) return fail(TOEP_ERR_INVALID, "ear %d out of range", ear);
  if (nyf < 1 || !yf || !out) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (r->dirs > 1 && out_pitch < nyf + r->g->length - 1) return fail(TOEP_ERR_INVALID, "output pitch too small");
  const int4* pairs = r->d_pairs ? r->d_pairs + (size_t)ear * r->pairs_per_ear * r->g->tap_stride : nullptr;
  const int4* pnnz = r->d_pnnz ? r->d_pnnz + (size_t)ear * r->pairs_per_ear : nullptr;
  return reflect_rows(r->g, ear * r->dirs, r->dirs, pairs, pnnz, yf, nyf, out, out_pitch, S(stream),
                      r->d_nonfinite);
}

}  // extern "C"

// ----------------------------------------------------------------- mixer ----
struct toep_mixer {
  const toep_renderer* r = nullptr;
  int S = 0;
  long long T = 0, zlen = 0;
  std::vector<int> h_dir;
  int order_s0 = -1, order_count = -1;  // source range the bucket tables describe
  int buckets = 0;
  int* d_bsrc = nullptr;  // sources sorted by direction
  int* d_bptr = nullptr;  // bucket b = d_bsrc[d_bptr[b] .. d_bptr[b+1])
  int* d_bdir = nullptr;  // direction of bucket b
  std::vector<int> h_bptr;
  unsigned long long* d_work = nullptr;  // k_mix item counter
  float* d_part = nullptr;
  size_t part_bytes = 0;
  // tensor-core path (mix_mma.cu): plan for the source range [mma_s0, mma_s0 + mma_count)
  bool mma = false;
  int N = 0, KP = 0, sexp = 20;
  int mma_s0 = -1, mma_count = -1, KS = 0, n_tiles = 0, ovh_pitch = 0, nsrc4 = 0, ring = 0;
  unsigned short* d_msrc = nullptr;
  int2* d_mks = nullptr;
  int* d_mrows = nullptr;
  float* d_mrowf = nullptr;
  unsigned char* d_mg = nullptr;
  float* d_ovh = nullptr;
  float* d_tmax = nullptr;
  int* d_bad = nullptr;  // [n_tiles] list + count + main-pass arrival counter
  std::vector<int2> h_taps;  // [rows][tap_stride] {offset, value bits}
  std::vector<int> h_nnz;
  const float* map_y = nullptr;  // source tensor map of the last call
  long long map_pitch = -1, map_rows = -1;
  CUtensorMap map{};
};

// TOEP_MIX_MMA=0 selects the FFMA/TMEM-window mix kernel (A/B runs)
static bool mix_mma_enabled() {
  const char* ev = getenv("TOEP_MIX_MMA");
  return !(ev && atoi(ev) == 0);
}

static void mma_plan_free(toep_mixer* m) {
  for (void* p : {(void*)m->d_msrc, (void*)m->d_mks, (void*)m->d_mrows, (void*)m->d_mrowf, (void*)m->d_mg,
                  (void*)m->d_ovh,
                  (void*)m->d_tmax, (void*)m->d_bad})
    if (p) cudaFree(p);
  m->d_msrc = nullptr;
  m->d_mks = nullptr;
  m->d_mrows = nullptr;
  m->d_mrowf = nullptr;
  m->d_mg = nullptr;
  m->d_ovh = nullptr;
  m->d_tmax = nullptr;
  m->d_bad = nullptr;
  m->mma_s0 = m->mma_count = -1;
}

static inline int mma_canon_host(int r, int k, int R) {
  return (k >> 4) * (R * 32) + (r >> 3) * 256 + ((k >> 3) & 1) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

// K-step plan of the tensor-core mix for sources [s0, s0+count): sources sorted
// by direction; a row = up to kMixRowSrcs sources of one direction; a K-step =
// up to 16 rows and kMixKsSrcs sources; G columns scaled per direction by
// 2^gamma_d (max |g_d| * 2^gamma_d in [2^13, 2^14)).
static int mma_plan(toep_mixer* m, int s0, int count, cudaStream_t st) {
  const toep_renderer* r = m->r;
  const toep_taps* g = r->g;
  if (m->h_taps.empty()) {
    m->h_taps.resize((size_t)g->rows * g->tap_stride);
    m->h_nnz.resize(g->rows);
    TOEP_CUDA(cudaMemcpyAsync(m->h_taps.data(), g->d_raw, m->h_taps.size() * sizeof(int2), cudaMemcpyDeviceToHost, st));
    TOEP_CUDA(cudaMemcpyAsync(m->h_nnz.data(), g->d_nnz, g->rows * sizeof(int), cudaMemcpyDeviceToHost, st));
    TOEP_CUDA(cudaStreamSynchronize(st));
  }
  mma_plan_free(m);
  const int* dir = m->h_dir.data() + s0;
  std::vector<int> ord(count);
  for (int i = 0; i < count; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [dir](int x, int y2) { return dir[x] < dir[y2]; });
  // rows: a direction's sources in groups of kMixRowSrcs, the remainder in one
  // smaller row.  Half K-steps hold 8 rows of ONE size class c (4, 3, 2, 1
  // sources), so a half is 8c consecutive ring slots, row r at [c r, c r + c)
  // (each builder warp takes one half: compile-time load offsets, no per-row
  // predicates); a K-step pairs two halves, classes c0 and c1, ks.y = n | c0 << 16
  // with n = 8 (c0 + c1) slots.  Only a class's last half has padding rows
  // (out-of-range source rows: TMA fills their slots with zeros, no memory
  // traffic), plus one padding half of class 1 when the count of halves is odd.
  struct Row { int d, first, cnt; };
  std::vector<Row> byc[kMixRowSrcs + 1];
  for (int p = 0; p < count;) {
    int q = p;
    while (q < count && dir[ord[q]] == dir[ord[p]]) ++q;
    for (int a2 = p; a2 < q; a2 += kMixRowSrcs) {
      const int c = std::min(kMixRowSrcs, q - a2);
      byc[c].push_back({dir[ord[p]], a2, c});
    }
    p = q;
  }
  // Rebalance the classes: splitting the e = (rows mod 8) rows of a class's
  // last, partly padded half into two smaller rows each (c = a + (c - a))
  // removes that half; keep a split when the modelled cost -- 40 slot loads
  // per K-step (MMAs, G stage, per-step builder work) + 1 per slot, padding
  // included -- drops.  Every source stays in exactly one row.
  {
    auto cost = [](const size_t* nr) {
      size_t halves = 0, slots = 0;
      for (int c = 1; c <= kMixRowSrcs; ++c) {
        halves += (nr[c] + 7) / 8;
        slots += (nr[c] + 7) / 8 * 8 * c;
      }
      if (halves & 1) slots += 8;
      return 40 * ((halves + 1) / 2) + slots;
    };
    for (;;) {
      size_t nr[kMixRowSrcs + 1];
      for (int c = 0; c <= kMixRowSrcs; ++c) nr[c] = byc[c].size();
      const size_t base = cost(nr);
      size_t best = base;
      int bc = 0, ba = 0;
      for (int c = 2; c <= kMixRowSrcs; ++c)
        for (int a = 1; 2 * a <= c; ++a) {
          const size_t e = nr[c] % 8;
          if (!e) continue;
          size_t t[kMixRowSrcs + 1];
          std::copy(nr, nr + kMixRowSrcs + 1, t);
          t[c] -= e;
          t[a] += e;
          t[c - a] += e;
          const size_t v = cost(t);
          if (v < best) {
            best = v;
            bc = c;
            ba = a;
          }
        }
      if (!bc) break;
      for (size_t e = byc[bc].size() % 8; e > 0; --e) {
        const Row w = byc[bc].back();
        byc[bc].pop_back();
        byc[ba].push_back({w.d, w.first, ba});
        byc[bc - ba].push_back({w.d, w.first + ba, bc - ba});
      }
    }
  }
  struct Half { int c; const Row* rows; int nr; };  // nr <= 8 real rows
  std::vector<Half> halves;
  for (int c = kMixRowSrcs; c >= 1; --c)
    for (size_t i = 0; i < byc[c].size(); i += 8)
      halves.push_back({c, byc[c].data() + i, (int)std::min<size_t>(8, byc[c].size() - i)});
  if (halves.size() & 1) halves.push_back({1, nullptr, 0});
  std::vector<int2> ks;
  std::vector<int> rinfo;    // [KS][16] (gamma_d + 128) << 9 (the fixup pass scales per row)
  std::vector<float> rowf;   // [KS][16] main-pass multipliers 2^(sexp - gamma_d)
  bool clamped = false;
  std::vector<int> ks_dirs;  // [KS][16] direction per row (-1 empty), gamma_d
  std::vector<unsigned short> src;  // K-step source lists: 8 rows x c0, then 8 rows x c1
  for (size_t hk = 0; hk < halves.size(); hk += 2) {
    const Half& h0 = halves[hk];
    const Half& h1 = halves[hk + 1];
    ks.push_back(make_int2((int)src.size(), (8 * (h0.c + h1.c)) | (h0.c << 16)));
    for (const Half* h : {&h0, &h1})
      for (int k = 0; k < 8; ++k)
        for (int u = 0; u < h->c; ++u) src.push_back((unsigned short)(k < h->nr ? ord[h->rows[k].first + u] : count));
    for (const Half* h : {&h0, &h1}) {
      for (int k = 0; k < 8; ++k) {
        if (k < h->nr) {
          const Row& w = h->rows[k];
          float mx = 0.f;
          for (int e = 0; e < r->ears; ++e) {
            const int row = e * r->dirs + w.d;
            for (int t = 0; t < m->h_nnz[row]; ++t) {
              float v;
              memcpy(&v, &m->h_taps[(size_t)row * g->tap_stride + t].y, 4);
              mx = std::max(mx, std::fabs(v));
            }
          }
          int gam = mx > 0.f ? 13 - std::ilogb(mx) : 0;
          gam = std::max(-126, std::min(126, gam));
          rinfo.push_back((gam + 128) << 9);
          const int em = m->sexp - gam;
          clamped |= em < -126 || em > 127;
          rowf.push_back(std::ldexp(1.f, std::max(-126, std::min(127, em))));
          ks_dirs.push_back(w.d);
          ks_dirs.push_back(gam);
        } else {
          rinfo.push_back(128 << 9);  // padding row
          rowf.push_back(0.f);
          ks_dirs.push_back(-1);
          ks_dirs.push_back(0);
        }
      }
    }
  }
  const int KS = (int)ks.size();
  const int N = m->N, KP = m->KP;
  const size_t gb = (size_t)N * 64;
  std::vector<unsigned char> G((size_t)KS * gb, 0);
  for (int k = 0; k < KS; ++k) {
    unsigned char* hi = G.data() + k * gb;
    unsigned char* lo = hi + gb / 2;
    for (int slot = 0; slot < 16; ++slot) {
      const int d = ks_dirs[(k * 16 + slot) * 2], gam = ks_dirs[(k * 16 + slot) * 2 + 1];
      if (d < 0) continue;
      for (int e = 0; e < r->ears; ++e) {
        const int row = e * r->dirs + d;
        for (int t = 0; t < m->h_nnz[row]; ++t) {
          const int2 tv = m->h_taps[(size_t)row * g->tap_stride + t];
          float v;
          memcpy(&v, &tv.y, 4);
          const float x = std::ldexp(v, gam);
          const __half h = __float2half_rn(x);
          const __half l = __float2half_rn(x - __half2float(h));
          const int off = mma_canon_host(e * KP + tv.x, slot, N);
          memcpy(hi + off, &h, 2);
          memcpy(lo + off, &l, 2);
        }
      }
    }
  }
  if (clamped) {  // a direction's gain is so far from the others that 2^(sexp - gamma) leaves fp32
    m->mma = false;
    return TOEP_OK;
  }
  m->KS = KS;
  m->nsrc4 = (int)src.size();
  m->ring = mix_mma_ring(N, r->ears, g->length, m->nsrc4, KS);
  if (m->ring == 0) {  // K-step tables too large for shared memory: take the FFMA mix
    m->mma = false;
    return TOEP_OK;
  }
  m->n_tiles = (int)((m->T + kMixTile - 1) / kMixTile);
  m->ovh_pitch = (int)std::max<long long>(4, round_up(g->length - 1, 4));
  cudaError_t e = cudaMalloc(&m->d_msrc, src.size() * sizeof(unsigned short));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_mks, KS * sizeof(int2));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_mrows, rinfo.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_mrowf, rowf.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_mg, G.size());
  if (e == cudaSuccess) e = cudaMalloc(&m->d_ovh, (size_t)m->n_tiles * r->ears * m->ovh_pitch * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_tmax, (size_t)m->n_tiles * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_bad, (size_t)(m->n_tiles + 2) * sizeof(int));
  if (e == cudaSuccess) e = cudaMemsetAsync(m->d_bad + m->n_tiles, 0, 2 * sizeof(int), st);  // count, arrivals
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(m->d_msrc, src.data(), src.size() * sizeof(unsigned short), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->d_mks, ks.data(), KS * sizeof(int2), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(m->d_mrows, rinfo.data(), rinfo.size() * sizeof(int), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(m->d_mg, G.data(), G.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(m->d_mrowf, rowf.data(), rowf.size() * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host staging vectors die here
  if (e != cudaSuccess) {
    mma_plan_free(m);
    return cuda_fail(e, "mixer tensor-core plan");
  }
  m->mma_s0 = s0;
  m->mma_count = count;
  return TOEP_OK;
}

static cudaError_t ensure_part(toep_mixer* m, size_t need, cudaStream_t st) {
  if (need <= m->part_bytes) return cudaSuccess;
  if (m->d_part) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    cudaFree(m->d_part);
    m->d_part = nullptr;
    m->part_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&m->d_part, need);
  if (e == cudaSuccess) m->part_bytes = need;
  return e;
}

extern "C" {

int toep_mixer_create(const toep_renderer* r, const int32_t* src_dir_host, int32_t n_src, int64_t T,
                      toep_mixer** out) {
  if (!out) return fail(TOEP_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (!r) return fail(TOEP_ERR_INVALID, "null renderer");
  if (n_src < 1 || !src_dir_host) return fail(TOEP_ERR_INVALID, "need at least one source");
  if (T < 1) return fail(TOEP_ERR_INVALID, "signal must be a non-empty 1-d array");
  if (r->g->kwin <= 0) return fail(TOEP_ERR_UNSUPPORTED, "mixdown supports reflection length <= 497");
  if (r->ears > 2) return fail(TOEP_ERR_UNSUPPORTED, "mixdown supports at most 2 ears");
  for (int s = 0; s < n_src; ++s)
    if (src_dir_host[s] < 0 || src_dir_host[s] >= r->dirs)  // engine/__init__.py:240-241
      return fail(TOEP_ERR_INVALID, "direction %d out of range", src_dir_host[s]);
  auto* m = new (std::nothrow) toep_mixer();
  if (!m) return fail(TOEP_ERR_NOMEM, "host allocation failed");
  m->r = r;
  m->S = n_src;
  m->T = T;
  m->zlen = T + r->g->length - 1;
  m->h_dir.assign(src_dir_host, src_dir_host + n_src);
  {
    const int K = r->g->length;
    m->KP = (int)round_up(K, 8);
    m->N = (int)round_up((long long)r->ears * m->KP, 16);
    const int ch = (K + 15) / 16, nr = (32 + K - 1 + 31) / 32;
    // overhang of one tile must stay within the next tile (K - 1 <= kMixTile)
    m->mma = mix_mma_enabled() && m->N <= 208 && K - 1 <= kMixTile && ((ch <= 7 && nr <= 5) || (ch <= 13 && nr <= 8));
    const char* se = getenv("TOEP_MIX_SEXP");
    if (se) m->sexp = std::max(-100, std::min(100, atoi(se)));
  }
  cudaError_t e = cudaMalloc(&m->d_bsrc, n_src * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_bptr, (n_src + 1) * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_bdir, n_src * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_work, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    toep_mixer_destroy(m);
    return cuda_fail(e, "toep_mixer_create");
  }
  *out = m;
  return TOEP_OK;
}

int toep_mixer_destroy(toep_mixer* m) {
  if (!m) return TOEP_OK;
  if (m->d_bsrc) cudaFree(m->d_bsrc);
  if (m->d_bptr) cudaFree(m->d_bptr);
  if (m->d_bdir) cudaFree(m->d_bdir);
  if (m->d_work) cudaFree(m->d_work);
  if (m->d_part) cudaFree(m->d_part);
  mma_plan_free(m);
  delete m;
  return TOEP_OK;
}

int64_t toep_mixer_z_len(const toep_mixer* m) { return m ? m->zlen : -1; }
int toep_mixer_path(const toep_mixer* m) { return m ? (m->mma ? TOEP_PATH_TENSOR : TOEP_PATH_WINDOW) : -1; }
// tensor path: main pass (its last CTA lists the fixup tiles), fixup pass,
// finish (overhang carry + z check); window path: mix, reduce, carry
int toep_mixer_kernels(const toep_mixer* m) { return m ? 3 : -1; }
int64_t toep_mixer_out_len(const toep_mixer* m) { return m ? m->zlen + m->r->lf - 1 : -1; }

int toep_mixer_partial(toep_mixer* m, const float* y, int64_t y_pitch, int32_t s0, int32_t count, float* z,
                       int64_t z_pitch, void* stream) {
  if (!m) return fail(TOEP_ERR_INVALID, "null mixer");
  if (count < 1 || s0 < 0 || (long long)s0 + count > m->S) return fail(TOEP_ERR_INVALID, "source range out of bounds");
  if (!y || !z) return fail(TOEP_ERR_INVALID, "null buffer");
  if (count > 1 && y_pitch < m->T) return fail(TOEP_ERR_INVALID, "source pitch too small");
  if ((reinterpret_cast<uintptr_t>(y) & 15) || (count > 1 && y_pitch % 4))
    return fail(TOEP_ERR_INVALID, "sources must be 16-byte aligned with a pitch multiple of 4");
  if (m->r->ears > 1 && z_pitch < m->zlen) return fail(TOEP_ERR_INVALID, "z pitch too small");
  cudaStream_t st = S(stream);
  const toep_taps* g = m->r->g;
  if (m->mma && count >= 65535) m->mma = false;  // K-step tables hold uint16 source rows
  if (m->mma && (s0 != m->mma_s0 || count != m->mma_count)) {
    const int rc = mma_plan(m, s0, count, st);  // may fall back to the FFMA mix (tables too large)
    if (rc != TOEP_OK) return rc;
  }
  if (m->mma) {
    MixMmaArgs a{};
    a.y = y;
    a.T = m->T;
    a.y_pitch = count > 1 ? y_pitch : round_up(m->T, 4);
    if (m->map_y != y || m->map_pitch != a.y_pitch || m->map_rows != count) {
      cudaError_t em = make_mix_source_map(y, m->T, count, a.y_pitch, &m->map);
      if (em != cudaSuccess) {
        m->map_y = nullptr;
        return cuda_fail(em, "tensor map (sources)");
      }
      m->map_y = y;
      m->map_pitch = a.y_pitch;
      m->map_rows = count;
    }
    a.src = m->d_msrc;
    a.ks = m->d_mks;
    a.rows = m->d_mrows;
    a.rowf = m->d_mrowf;
    a.g = m->d_mg;
    a.KS = m->KS;
    a.nsrc4 = m->nsrc4;
    a.ring = m->ring;
    a.N = m->N;
    a.KP = m->KP;
    a.K = g->length;
    a.ears = m->r->ears;
    a.n_tiles = m->n_tiles;
    a.sexp = m->sexp;
    a.z = z;
    a.z_pitch = m->r->ears > 1 ? z_pitch : 0;
    a.zlen = m->zlen;
    a.ovh = m->d_ovh;
    a.ovh_pitch = m->ovh_pitch;
    a.tile_max = m->d_tmax;
    a.nonfinite = m->r->d_nonfinite;
    cudaError_t e = launch_mix_mma(a, m->map, m->d_bad, m->d_bad + m->n_tiles, sm_count_cached(), st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_mix_mma");
    return TOEP_OK;
  }
  if (s0 != m->order_s0 || count != m->order_count) {
    // buckets: stable sort of the range by direction; bucket b = sources
    // bsrc[bptr[b] .. bptr[b+1]) (indices relative to s0), all at bdir[b]
    std::vector<int> ord(count);
    for (int i = 0; i < count; ++i) ord[i] = i;
    const int* dir = m->h_dir.data() + s0;
    std::stable_sort(ord.begin(), ord.end(), [dir](int x, int y2) { return dir[x] < dir[y2]; });
    std::vector<int> bptr(1, 0), bdir;  // a direction with more than kMixGroupSrcCap sources spans several buckets
    for (int p = 0; p < count; ++p) {
      if (p + 1 == count || dir[ord[p + 1]] != dir[ord[p]] || p + 1 - bptr.back() == kMixGroupSrcCap) {
        bdir.push_back(dir[ord[p]]);
        bptr.push_back(p + 1);
      }
    }
    m->buckets = (int)bdir.size();
    m->h_bptr = bptr;
    TOEP_CUDA(cudaMemcpyAsync(m->d_bsrc, ord.data(), count * sizeof(int), cudaMemcpyHostToDevice, st));
    TOEP_CUDA(cudaMemcpyAsync(m->d_bptr, bptr.data(), bptr.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    TOEP_CUDA(cudaMemcpyAsync(m->d_bdir, bdir.data(), bdir.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    TOEP_CUDA(cudaStreamSynchronize(st));
    m->order_s0 = s0;
    m->order_count = count;
  }
  const int n_tiles = (int)((m->zlen + kW - 1) / kW);
  const long long part_pitch = (long long)n_tiles * kW;
  // one pass: the mix kernel sums each bucket's sources per tile on the fly
  {
    const int sm = sm_count_cached();
    const long long slots = (long long)sm * (512 / (kR + g->kwin));
    // >= ~24 items per persistent CTA keeps the tail short; fewer groups keep the partials small
    const long long ipc = 24;  // items per CTA (12 / 48 / 96 measured no better)
    long long bpg = ((long long)m->buckets * n_tiles + ipc * slots - 1) / (ipc * slots);
    bpg = std::max(16LL, std::min<long long>(std::min<long long>(bpg, kMixMaxBuckets), m->buckets));
    auto group_srcs = [&](long long per) {  // largest source count of a group of `per` buckets
      int g = 0;
      for (long long b0 = 0; b0 < m->buckets; b0 += per)
        g = std::max(g, m->h_bptr[std::min<long long>(b0 + per, m->buckets)] - m->h_bptr[b0]);
      return g;
    };
    int gsrc = group_srcs(bpg);
    while (gsrc > kMixGroupSrcCap && bpg > 1) gsrc = group_srcs(bpg = (bpg + 1) / 2);  // the tables live in smem
    const int groups = (int)((m->buckets + bpg - 1) / bpg);
    TOEP_CUDA(ensure_part(m, (size_t)groups * m->r->ears * part_pitch * sizeof(float), st));
    MixArgs a{};
    a.y = y;
    a.T = m->T;
    a.y_pitch = count > 1 ? y_pitch : round_up(m->T, 4);
    a.bsrc = m->d_bsrc;
    a.bptr = m->d_bptr;
    a.bdir = m->d_bdir;
    a.buckets = m->buckets;
    a.buckets_per_group = (int)bpg;
    a.group_srcs = (gsrc + 3) & ~3;
    a.groups = groups;
    a.n_tiles = n_tiles;
    a.n_items = (long long)groups * n_tiles;
    a.taps = g->d_kw;
    a.etaps = m->r->d_epairs;
    a.row_nnz = g->d_nnz;
    a.tap_stride = g->tap_stride;
    a.dirs = m->r->dirs;
    a.ears = m->r->ears;
    a.part = m->d_part;
    a.part_pitch = part_pitch;
    a.zlen = m->zlen;
    a.nonfinite = m->r->d_nonfinite;
    a.work = m->d_work;
    TOEP_CUDA(cudaMemsetAsync(m->d_work, 0, sizeof(unsigned long long), st));
    cudaError_t e = launch_mix(a, g->kwin, g->uniform ? g->max_nnz : 0, sm, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_mix");
    e = launch_mix_reduce(m->d_part, groups, m->r->ears, part_pitch, m->zlen, z, z_pitch, st);
    if (e != cudaSuccess) return cuda_fail(e, "launch_mix_reduce");
    return TOEP_OK;
  }
}

int toep_mixer_finish(const toep_mixer* m, const float* z, int64_t z_pitch, float* out, int64_t out_pitch,
                      void* stream) {
  if (!m) return fail(TOEP_ERR_INVALID, "null mixer");
  if (!z || !out) return fail(TOEP_ERR_INVALID, "null buffer");
  const long long out_len = toep_mixer_out_len(m);
  if (m->r->ears > 1 && out_pitch < out_len) return fail(TOEP_ERR_INVALID, "output pitch too small");
  return dense_fir(z, m->zlen, z_pitch, m->r->d_f, m->r->lf_pad, m->r->lf_pad, m->r->ears, out, out_len, out_pitch,
                   S(stream));
}

}  // extern "C"

// -------------------------------------------------------------- streamer ----
struct toep_streamer {
  const toep_renderer* r = nullptr;
  int S = 0, B = 0, H = 0, zh = 0, ctas = 0, spc = 0, nzh = 0, ntk = 0;
  bool cluster = true;
  int* d_dir = nullptr;
  int2* d_srctaps = nullptr;  // [S][ears][tap_stride]
  int* d_srcnnz = nullptr;    // [S][ears]
  float* d_yhist = nullptr;
  float* d_zhist = nullptr;   // [groups][ears][zh]
  float* d_part = nullptr;
  float* d_gpart = nullptr;
  unsigned int* d_ticket = nullptr;
};

extern "C" {

int toep_streamer_create(const toep_renderer* r, const int32_t* src_dir_host, int32_t n_src, int32_t block,
                         toep_streamer** out) {
  if (!out) return fail(TOEP_ERR_INVALID, "null output handle");
  *out = nullptr;
  if (!r) return fail(TOEP_ERR_INVALID, "null renderer");
  if (n_src < 1 || !src_dir_host) return fail(TOEP_ERR_INVALID, "need at least one source");
  if (block < 4 || block > 256 || block % 4) return fail(TOEP_ERR_UNSUPPORTED, "block size must be a multiple of 4 in [4, 256]");
  if (r->ears > 2) return fail(TOEP_ERR_UNSUPPORTED, "streaming supports at most 2 ears");
  if (r->g->length > 4096) return fail(TOEP_ERR_UNSUPPORTED, "streaming supports reflection length <= 4096");
  for (int s = 0; s < n_src; ++s)
    if (src_dir_host[s] < 0 || src_dir_host[s] >= r->dirs)
      return fail(TOEP_ERR_INVALID, "direction %d out of range", src_dir_host[s]);
  auto* s = new (std::nothrow) toep_streamer();
  if (!s) return fail(TOEP_ERR_NOMEM, "host allocation failed");
  s->r = r;
  s->S = n_src;
  s->B = block;
  s->H = (int)round_up(std::max(1, r->g->length - 1), 4);
  s->zh = r->lf_pad;
  // 4 sources per CTA: ~1 CTA per SM for 512 sources, short per-thread tap chains
  // sources per CTA: 4 (the two-level kernel), 2 for the cluster kernel (its
  // exchange is cheap, so more CTAs shorten the source phase: 11.1 vs 11.6 us
  // per cfg4 block); bounded by the 96 KB of windows + taps per CTA
  s->cluster = stream_cluster_enabled();
  s->spc = std::max(1, std::min(s->cluster ? 2 : 4,
                                (96 * 1024 / 4) / (s->H + block + 2 * r->ears * ((r->g->tap_stride + 7) / 8 * 8) + r->ears)));
  if (const char* ev = getenv("TOEP_STREAM_SPC")) s->spc = std::max(1, std::min(s->spc, atoi(ev)));  // A/B runs
  s->ctas = stream_ctas(n_src, s->spc, s->cluster);
  // z-history sets and tickets for either streaming kernel: groups of
  // k_stream_step or clusters of k_stream_cl
  s->nzh = std::max((s->ctas + kStreamGroup - 1) / kStreamGroup, (s->ctas + kStreamCL - 1) / kStreamCL);
  s->ntk = std::max(s->nzh + 1, kStreamCL);
  const int groups = s->nzh;
  cudaError_t e = cudaMalloc(&s->d_dir, n_src * sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpy(s->d_dir, src_dir_host, n_src * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_yhist, (size_t)n_src * s->H * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_zhist, (size_t)groups * r->ears * s->zh * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_srctaps, (size_t)n_src * r->ears * r->g->tap_stride * sizeof(int2));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_srcnnz, (size_t)n_src * r->ears * sizeof(int));
  if (e == cudaSuccess)
    e = launch_stream_gather_taps(r->g->d_raw, r->g->d_nnz, s->d_dir, n_src, r->ears, r->dirs, r->g->tap_stride,
                                  s->d_srctaps, s->d_srcnnz, nullptr);
  if (e == cudaSuccess) e = cudaMalloc(&s->d_part, (size_t)s->ctas * r->ears * block * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_gpart, (size_t)groups * r->ears * block * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->d_ticket, s->ntk * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(s->d_yhist, 0, (size_t)n_src * s->H * sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(s->d_zhist, 0, (size_t)groups * r->ears * s->zh * sizeof(float));
  if (e == cudaSuccess) e = cudaMemset(s->d_ticket, 0, s->ntk * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    toep_streamer_destroy(s);
    return cuda_fail(e, "toep_streamer_create");
  }
  *out = s;
  return TOEP_OK;
}

int toep_streamer_destroy(toep_streamer* s) {
  if (!s) return TOEP_OK;
  if (s->d_dir) cudaFree(s->d_dir);
  if (s->d_srctaps) cudaFree(s->d_srctaps);
  if (s->d_srcnnz) cudaFree(s->d_srcnnz);
  if (s->d_yhist) cudaFree(s->d_yhist);
  if (s->d_zhist) cudaFree(s->d_zhist);
  if (s->d_part) cudaFree(s->d_part);
  if (s->d_gpart) cudaFree(s->d_gpart);
  if (s->d_ticket) cudaFree(s->d_ticket);
  delete s;
  return TOEP_OK;
}

int toep_streamer_reset(toep_streamer* s, void* stream) {
  if (!s) return fail(TOEP_ERR_INVALID, "null streamer");
  cudaStream_t st = S(stream);
  TOEP_CUDA(cudaMemsetAsync(s->d_yhist, 0, (size_t)s->S * s->H * sizeof(float), st));
  TOEP_CUDA(cudaMemsetAsync(s->d_zhist, 0, (size_t)s->nzh * s->r->ears * s->zh * sizeof(float), st));
  TOEP_CUDA(cudaMemsetAsync(s->d_ticket, 0, s->ntk * sizeof(unsigned int), st));
  return TOEP_OK;
}

int toep_streamer_step(toep_streamer* s, const float* block, int64_t block_pitch, float* out, int64_t out_pitch,
                       void* stream) {
  if (!s) return fail(TOEP_ERR_INVALID, "null streamer");
  if (!block || !out) return fail(TOEP_ERR_INVALID, "null buffer");
  if (s->S > 1 && block_pitch < s->B) return fail(TOEP_ERR_INVALID, "block pitch too small");
  if ((reinterpret_cast<uintptr_t>(block) & 15) || (s->S > 1 && block_pitch % 4))
    return fail(TOEP_ERR_INVALID, "block must be 16-byte aligned with a pitch multiple of 4");
  if (s->r->ears > 1 && out_pitch < s->B) return fail(TOEP_ERR_INVALID, "output pitch too small");
  StreamArgs a{};
  a.block = block;
  a.block_pitch = s->S > 1 ? block_pitch : s->B;
  a.B = s->B;
  a.yhist = s->d_yhist;
  a.H = s->H;
  a.S = s->S;
  a.src_taps = s->d_srctaps;
  a.src_nnz = s->d_srcnnz;
  a.tap_stride = s->r->g->tap_stride;
  a.ears = s->r->ears;
  a.src_per_cta = s->spc;
  a.part = s->d_part;
  a.gpart = s->d_gpart;
  a.zhist = s->d_zhist;
  a.zh = s->zh;
  a.f = s->r->d_f;
  a.lf_pad = s->r->lf_pad;
  a.out = out;
  a.out_pitch = s->r->ears > 1 ? out_pitch : s->B;
  a.ctas = s->ctas;
  a.ticket = s->d_ticket;
  a.nonfinite = s->r->d_nonfinite;
  a.cluster = s->cluster ? 1 : 0;
  cudaError_t e = launch_stream_step(a, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "launch_stream_step");
  return TOEP_OK;
}

}  // extern "C"
