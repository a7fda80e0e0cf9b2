// Radix-2 FFT and FFT overlap-save convolution (the engine's third mode).
//
// Reference semantics:
//   fft(data, bitrev, twiddles, inverse)         _kernels.pyx:47-77  (iterative radix-2,
//       bit-reversed load, decimation in time, inverse scaled by 1/n; macs = butterflies)
//   _overlap_save(plan, y, kernels)               engine/__init__.py:178-205 (blocks of n
//       samples advancing by n - ntaps + 1, product with the taps' spectrum, inverse,
//       keep samples [ntaps-1, n))
//
// Kernels:
//   k_fft_smem     one transform per CTA in shared memory (bit-reversed gather from
//                  global, log2(n) in-place DIT stages, one barrier per stage);
//                  complex128 for the plugin `fft` (the reference's precision),
//                  complex64 inside the convolution
//   k_fft_stage    one radix-2 stage over global memory, batched (transforms larger
//                  than shared memory)
//   k_ols_fused    overlap-save for blocks <= kOlsSmemMax: a CTA per block does gather,
//                  forward FFT, spectrum product, in-shared-memory bit reversal,
//                  inverse FFT and the store of the valid samples in one pass
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "common.cuh"
#include "launch.h"

namespace toep {

template <typename T>
struct Cplx;
template <>
struct Cplx<float> {
  using T2 = float2;
};
template <>
struct Cplx<double> {
  using T2 = double2;
};

template <typename T2>
__device__ __forceinline__ T2 cmul(T2 a, T2 b) {
  T2 r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}

__device__ __forceinline__ unsigned bitrev(unsigned i, int logn) { return logn ? __brev(i) >> (32 - logn) : 0u; }

// In-place DIT stages over a bit-reversed shared buffer; tw[k] = exp(-2 pi i k / n), k < n/2.
template <typename T2, bool INV>
__device__ __forceinline__ void fft_stages_smem(T2* a, const T2* __restrict__ tw, int n, int logn) {
  for (int s = 1; s <= logn; ++s) {
    const int half = 1 << (s - 1);
    const int tstride = n >> s;  // twiddle index step
    for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
      const int grp = b >> (s - 1), k = b & (half - 1);
      const int i0 = (grp << s) + k, i1 = i0 + half;
      T2 w = tw[k * tstride];
      if (INV) w.y = -w.y;
      const T2 u = a[i0];
      const T2 v = cmul(w, a[i1]);
      a[i0] = T2{u.x + v.x, u.y + v.y};
      a[i1] = T2{u.x - v.x, u.y - v.y};
    }
    __syncthreads();
  }
}

template <typename T, bool INV>
__global__ void k_fft_smem(const typename Cplx<T>::T2* __restrict__ in, typename Cplx<T>::T2* __restrict__ out,
                           const typename Cplx<T>::T2* __restrict__ tw, int n, int logn) {
  using T2 = typename Cplx<T>::T2;
  extern __shared__ __align__(16) unsigned char smem_fft[];
  T2* a = reinterpret_cast<T2*>(smem_fft);
  const T2* src = in + (long long)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[bitrev(i, logn)] = src[i];
  __syncthreads();
  fft_stages_smem<T2, INV>(a, tw, n, logn);
  T2* dst = out + (long long)blockIdx.x * n;
  const T scale = INV ? T(1) / T(n) : T(1);
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = T2{a[i].x * scale, a[i].y * scale};
}

template <typename T>
__global__ void k_fft_bitrev(const typename Cplx<T>::T2* __restrict__ in, typename Cplx<T>::T2* __restrict__ out,
                             long long n, int logn, long long total) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x) {
    const long long b = g >> logn, i = g & (n - 1);
    const unsigned long long r = logn ? __brevll((unsigned long long)i) >> (64 - logn) : 0ull;
    out[b * n + (long long)r] = in[g];
  }
}

template <typename T, bool INV>
__global__ void k_fft_stage(typename Cplx<T>::T2* __restrict__ a, const typename Cplx<T>::T2* __restrict__ tw,
                            long long n, int s, long long total_bf, T scale) {
  using T2 = typename Cplx<T>::T2;
  const long long half = 1LL << (s - 1), tstride = n >> s;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total_bf; g += (long long)gridDim.x * blockDim.x) {
    const long long b = g / (n / 2), bf = g - b * (n / 2);
    const long long grp = bf >> (s - 1), k = bf & (half - 1);
    T2* x = a + b * n;
    const long long i0 = (grp << s) + k, i1 = i0 + half;
    T2 w = tw[k * tstride];
    if (INV) w.y = -w.y;
    const T2 u = x[i0];
    const T2 v = cmul(w, x[i1]);
    x[i0] = T2{(u.x + v.x) * scale, (u.y + v.y) * scale};
    x[i1] = T2{(u.x - v.x) * scale, (u.y - v.y) * scale};
  }
}

// Overlap-save, one CTA per block of n samples (n <= kOlsSmemMax): segment
// b = stream[b*valid, b*valid + n), stream = [0 x (ntaps-1), y, 0 ...].
__global__ void k_ols_fused(const float* __restrict__ y, long long ny, const float2* __restrict__ spec,
                            const float2* __restrict__ tw, int n, int logn, int ntaps, float* __restrict__ out,
                            long long out_len) {
  extern __shared__ __align__(16) unsigned char smem_fft[];
  float2* a = reinterpret_cast<float2*>(smem_fft);
  const int valid = n - ntaps + 1;
  const long long s0 = (long long)blockIdx.x * valid - (ntaps - 1);  // y index of segment[0]
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const long long t = s0 + i;
    a[bitrev(i, logn)] = make_float2((t >= 0 && t < ny) ? __ldg(y + t) : 0.f, 0.f);
  }
  __syncthreads();
  fft_stages_smem<float2, false>(a, tw, n, logn);
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = cmul(a[i], spec[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {  // in-place bit reversal for the inverse DIT
    const int r = (int)bitrev(i, logn);
    if (r > i) {
      const float2 tmp = a[i];
      a[i] = a[r];
      a[r] = tmp;
    }
  }
  __syncthreads();
  fft_stages_smem<float2, true>(a, tw, n, logn);
  const float scale = 1.f / (float)n;
  for (int i = threadIdx.x; i < valid; i += blockDim.x) {
    const long long t = (long long)blockIdx.x * valid + i;
    if (t < out_len) out[t] = a[ntaps - 1 + i].x * scale;
  }
}

// overlap-save helpers for large blocks: gather segments, spectrum product, extract
__global__ void k_ols_gather(const float* __restrict__ y, long long ny, float2* __restrict__ seg, int n, int ntaps,
                             long long total) {
  const int valid = n - ntaps + 1;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x) {
    const long long b = g / n, i = g - b * n;
    const long long t = b * valid - (ntaps - 1) + i;
    seg[g] = make_float2((t >= 0 && t < ny) ? __ldg(y + t) : 0.f, 0.f);
  }
}

__global__ void k_ols_product(float2* __restrict__ seg, const float2* __restrict__ spec, int n, long long total) {
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x)
    seg[g] = cmul(seg[g], spec[g % n]);
}

__global__ void k_ols_extract(const float2* __restrict__ seg, int n, int ntaps, float* __restrict__ out,
                              long long out_len) {
  const int valid = n - ntaps + 1;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < out_len; t += (long long)gridDim.x * blockDim.x) {
    const long long b = t / valid, i = t - b * valid;
    out[t] = seg[b * n + ntaps - 1 + i].x;
  }
}

__global__ void k_pack_real(const float* __restrict__ x, long long nx, float2* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = make_float2(i < nx ? x[i] : 0.f, 0.f);
}

// ---------------------------------------------------------------- host ----
// Twiddle tables exp(-2 pi i k / n), k < n/2, computed in double on the host,
// cached per (device, n, precision) for the process lifetime.
static std::mutex g_tw_mu;
static std::unordered_map<long long, void*> g_tw;

static cudaError_t twiddles(long long n, bool dbl, const void** out) {
  int dev = 0;
  cudaError_t ed = cudaGetDevice(&dev);
  if (ed != cudaSuccess) return ed;
  std::lock_guard<std::mutex> lk(g_tw_mu);
  const long long key = ((long long)dev << 48) | (n * 2 + (dbl ? 1 : 0));
  auto it = g_tw.find(key);
  if (it != g_tw.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  const long long h = std::max(1LL, n / 2);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, h * (dbl ? sizeof(double2) : sizeof(float2)));
  if (e != cudaSuccess) return e;
  if (dbl) {
    std::vector<double2> w(h);
    for (long long k = 0; k < h; ++k) {
      const double ang = -2.0 * M_PI * (double)k / (double)n;
      w[k] = make_double2(std::cos(ang), std::sin(ang));
    }
    e = cudaMemcpy(d, w.data(), h * sizeof(double2), cudaMemcpyHostToDevice);
  } else {
    std::vector<float2> w(h);
    for (long long k = 0; k < h; ++k) {
      const double ang = -2.0 * M_PI * (double)k / (double)n;
      w[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
    e = cudaMemcpy(d, w.data(), h * sizeof(float2), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(d);
    return e;
  }
  g_tw[key] = d;
  *out = d;
  return cudaSuccess;
}

static int ilog2(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

constexpr long long kFftSmemBytes = 128 * 1024;  // one transform in shared memory up to this size

template <typename T>
static cudaError_t fft_batched(const typename Cplx<T>::T2* in, typename Cplx<T>::T2* out, long long n,
                               long long batch, bool inverse, cudaStream_t st) {
  using T2 = typename Cplx<T>::T2;
  const void* twv = nullptr;
  cudaError_t e = twiddles(n, sizeof(T) == 8, &twv);
  if (e != cudaSuccess) return e;
  const T2* tw = reinterpret_cast<const T2*>(twv);
  const int logn = ilog2(n);
  if (n * (long long)sizeof(T2) <= kFftSmemBytes) {
    const int bytes = (int)(n * sizeof(T2));
    const int threads = (int)std::min<long long>(512, std::max<long long>(32, n / 2));
    auto kern = inverse ? k_fft_smem<T, true> : k_fft_smem<T, false>;
    if (bytes > 48 * 1024) {
      e = ensure_smem(reinterpret_cast<const void*>(kern), bytes);
      if (e != cudaSuccess) return e;
    }
    kern<<<(unsigned)batch, threads, bytes, st>>>(in, out, tw, (int)n, logn);
    return cudaGetLastError();
  }
  const long long total = n * batch;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  k_fft_bitrev<T><<<blocks, 256, 0, st>>>(in, out, n, logn, total);
  const long long bfs = total / 2;
  const int bb = (int)std::min<long long>((bfs + 255) / 256, 148 * 32);
  for (int s = 1; s <= logn; ++s) {
    const T scale = (inverse && s == logn) ? T(1) / T(n) : T(1);
    if (inverse)
      k_fft_stage<T, true><<<bb, 256, 0, st>>>(out, tw, n, s, bfs, scale);
    else
      k_fft_stage<T, false><<<bb, 256, 0, st>>>(out, tw, n, s, bfs, scale);
  }
  return cudaGetLastError();
}

cudaError_t launch_fft_c128(const double* in, double* out, long long n, bool inverse, cudaStream_t st) {
  return fft_batched<double>(reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out), n, 1, inverse, st);
}

cudaError_t launch_fft_c64(const float* in, float* out, long long n, long long batch, bool inverse, cudaStream_t st) {
  return fft_batched<float>(reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), n, batch, inverse, st);
}

cudaError_t launch_fft_conv(const float* y, long long ny, const float* spectrum, long long n, long long ntaps,
                            float* out, float* scratch, cudaStream_t st) {
  const long long valid = n - ntaps + 1;
  const long long out_len = ny + ntaps - 1;
  const long long nseg = (out_len + valid - 1) / valid;
  const void* twv = nullptr;
  cudaError_t e = twiddles(n, false, &twv);
  if (e != cudaSuccess) return e;
  const float2* tw = reinterpret_cast<const float2*>(twv);
  const float2* spec = reinterpret_cast<const float2*>(spectrum);
  if (n * (long long)sizeof(float2) <= kFftSmemBytes) {
    const int bytes = (int)(n * sizeof(float2));
    const int threads = (int)std::min<long long>(512, std::max<long long>(32, n / 2));
    if (bytes > 48 * 1024) {
      e = ensure_smem(reinterpret_cast<const void*>(k_ols_fused), bytes);
      if (e != cudaSuccess) return e;
    }
    k_ols_fused<<<(unsigned)nseg, threads, bytes, st>>>(y, ny, spec, tw, (int)n, ilog2(n), (int)ntaps, out, out_len);
    return cudaGetLastError();
  }
  // large blocks: segments through global memory, ping-pong between the two
  // halves of scratch (the bit-reversal pass of the global FFT is out of place)
  const long long total = nseg * n;
  float2* segA = reinterpret_cast<float2*>(scratch);
  float2* segB = segA + total;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  k_ols_gather<<<blocks, 256, 0, st>>>(y, ny, segA, (int)n, (int)ntaps, total);
  e = fft_batched<float>(segA, segB, n, nseg, false, st);
  if (e != cudaSuccess) return e;
  k_ols_product<<<blocks, 256, 0, st>>>(segB, spec, (int)n, total);
  e = fft_batched<float>(segB, segA, n, nseg, true, st);
  if (e != cudaSuccess) return e;
  const int ob = (int)std::min<long long>((out_len + 255) / 256, 148 * 32);
  k_ols_extract<<<ob, 256, 0, st>>>(segA, (int)n, (int)ntaps, out, out_len);
  return cudaGetLastError();
}

// spectrum[n] (complex64) = DFT of the taps zero-padded to n; tmp holds n complex64
cudaError_t launch_fft_spectrum(const float* taps, long long ntaps, long long n, float* spectrum, float* tmp,
                                cudaStream_t st) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 1024);
  k_pack_real<<<blocks, 256, 0, st>>>(taps, ntaps, reinterpret_cast<float2*>(tmp), n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return fft_batched<float>(reinterpret_cast<const float2*>(tmp), reinterpret_cast<float2*>(spectrum), n, 1, false, st);
}

long long fft_conv_scratch_bytes(long long ny, long long n, long long ntaps) {
  if (n * (long long)sizeof(float2) <= kFftSmemBytes) return 0;
  const long long valid = n - ntaps + 1, out_len = ny + ntaps - 1;
  return 2 * ((out_len + valid - 1) / valid) * n * (long long)sizeof(float2);
}

// transforms larger than shared memory need distinct in/out buffers
bool fft_needs_distinct(long long n, bool dbl) {
  return n * (long long)(dbl ? sizeof(double2) : sizeof(float2)) > kFftSmemBytes;
}

}  // namespace toep
