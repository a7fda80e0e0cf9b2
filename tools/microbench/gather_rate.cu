// Load-side probe for a tensor-core mixdown: how fast can one persistent CTA
// per SM pull every source's slice of a time tile into shared memory when the
// sources arrive in bucket (direction) order, i.e. as random rows of the
// [S][T] source array?  (config 5: 4,096 x 2,880,000 fp32 = 47 GB.)
//
// Per tile of TW samples the CTA walks all S sources in stages of GS slices;
// a producer fills a STAGES-deep shared-memory ring, CW consumer warps sum
// each stage into per-thread registers (stand-in for the direction sums) and
// release the slot.  Producers:
//   bulk    : one elected thread, one cp.async.bulk (1-D TMA) per slice
//   ldgsts  : P producer warps, cp.async 16 B per lane, completion through
//             cp.async.mbarrier.arrive.noinc
//   gather4 : one elected thread, one 2-D tensor TMA tile::gather4 per 4 slices
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_rate gather_rate.cu -lcuda
//   ./gather_rate [T]
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);                \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::
          "r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  unsigned p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(p));
  return p != 0;
}

__global__ void k_init(float* y, int S, long long pitch) {
  const long long n = (long long)S * pitch;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long s = i / pitch, t = i - s * pitch;
    y[i] = (float)(((s * 7 + t) % 5) - 2);
  }
}

template <int MODE, int TW, int GS, int STAGES, int CW, int PW>
__global__ void __launch_bounds__(32 * (CW + PW), 1)
    k_gather(const float* __restrict__ y, long long pitch, const int* __restrict__ order, int S, int ntiles,
             float* __restrict__ out, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(128) unsigned char smraw[];
  float* ring = reinterpret_cast<float*>(smraw);  // [STAGES][GS][TW]
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + STAGES * GS * TW * 4);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], MODE == 1 ? 32 * PW : 1);
      mbar_init(&empty[i], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int ngroups = S / GS;
  const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x), t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
  if (warp >= CW) {  // producers
    const int pw = warp - CW;
    int st = 0;
    unsigned ph = 0;
    for (int tile = t0; tile < t1; ++tile) {
      for (int g = 0; g < ngroups; ++g) {
        mbar_wait(&empty[st], ph ^ 1u);
        float* dst = ring + st * GS * TW;
        if (MODE == 0) {
          if (pw == 0 && elect_one()) {
            mbar_expect(&full[st], GS * TW * 4);
            for (int u = 0; u < GS; ++u) {
              const float* src = y + (long long)order[g * GS + u] * pitch + (long long)tile * TW;
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      su32(dst + u * TW)),
                  "l"(src), "r"(TW * 4), "r"(su32(&full[st]))
                  : "memory");
            }
          }
        } else if (MODE == 1) {
          constexpr int C16 = TW / 4;  // 16-byte chunks per slice
          for (int u = pw; u < GS; u += PW) {
            const float* src = y + (long long)order[g * GS + u] * pitch + (long long)tile * TW;
            for (int c = lane; c < C16; c += 32)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + u * TW + 4 * c)),
                           "l"(src + 4 * c)
                           : "memory");
          }
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
        } else {
          if (pw == 0 && elect_one()) {
            mbar_expect(&full[st], GS * TW * 4);
            for (int u = 0; u < GS; u += 4) {
              const int* o = order + g * GS + u;
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, "
                  "{%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst + u * TW)),
                  "l"(&tm), "r"(tile * TW), "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(su32(&full[st]))
                  : "memory");
            }
          }
        }
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    }
  } else {  // consumers: thread owns TW / (32 CW) time columns
    constexpr int PER = TW / (32 * CW);
    int st = 0;
    unsigned ph = 0;
    for (int tile = t0; tile < t1; ++tile) {
      float acc[PER > 0 ? PER : 1];
#pragma unroll
      for (int i = 0; i < PER; ++i) acc[i] = 0.f;
      for (int g = 0; g < ngroups; ++g) {
        mbar_wait(&full[st], ph);
        const float* src = ring + st * GS * TW;
#pragma unroll 4
        for (int u = 0; u < GS; ++u)
#pragma unroll
          for (int i = 0; i < PER; ++i) acc[i] += src[u * TW + threadIdx.x + 32 * CW * i];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) out[(long long)tile * TW + threadIdx.x + 32 * CW * i] = acc[i];
    }
  }
}

template <int MODE, int TW, int GS, int STAGES, int CW, int PW>
static void run(const char* name, EncodeTiledFn enc, float* y, long long pitch, long long T, int* d_order, int S,
                float* out, int sms, const std::vector<float>& ref_sum) {
  const int ntiles = (int)(T / TW);
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  if (MODE == 2) {
    const cuuint64_t dims[2] = {(cuuint64_t)T, (cuuint64_t)S};
    const cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    const cuuint32_t box[2] = {TW, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%-40s encode failed (%d)\n", name, (int)r);
      return;
    }
  }
  auto kern = k_gather<MODE, TW, GS, STAGES, CW, PW>;
  const int smem = STAGES * GS * TW * 4 + 2 * STAGES * 8;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  kern<<<sms, 32 * (CW + PW), smem>>>(y, pitch, d_order, S, ntiles, out, tm);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(a));
    kern<<<sms, 32 * (CW + PW), smem>>>(y, pitch, d_order, S, ntiles, out, tm);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  // check a few tile sums
  std::vector<float> h(4096);
  CK(cudaMemcpy(h.data(), out, 4096 * 4, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < 4096 && i < (int)ref_sum.size(); ++i) err = std::max(err, (double)fabsf(h[i] - ref_sum[i]));
  const double bytes = (double)S * ntiles * TW * 4;
  printf("%-40s %8.3f ms  %7.1f GB/s  (max err %.2e)\n", name, best, bytes / best / 1e6, err);
}

int main(int argc, char** argv) {
  const long long T = argc > 1 ? atoll(argv[1]) : 2880000LL;
  const int S = 4096;
  const long long pitch = (T + 3) / 4 * 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* y;
  CK(cudaMalloc(&y, (size_t)S * pitch * 4));
  // y[s][t] = small integers so sums are exact: ((s * 7 + t) % 5) - 2
  k_init<<<4096, 256>>>(y, S, pitch);
  CK(cudaDeviceSynchronize());
  std::vector<int> order(S);
  std::iota(order.begin(), order.end(), 0);
  std::mt19937 rng(5);
  std::shuffle(order.begin(), order.end(), rng);
  int* d_order;
  CK(cudaMalloc(&d_order, S * 4));
  CK(cudaMemcpy(d_order, order.data(), S * 4, cudaMemcpyHostToDevice));
  float* out;
  CK(cudaMalloc(&out, (size_t)pitch * 4));
  std::vector<float> ref(4096);
  for (int t = 0; t < 4096; ++t) {
    double s = 0;
    for (int u = 0; u < S; ++u) s += ((u * 7 + t) % 5) - 2;
    ref[t] = (float)s;
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeTiledFn enc = (EncodeTiledFn)fn;
  printf("S=%d T=%lld (%.2f GB), %d SMs\n", S, T, (double)S * T * 4 / 1e9, sms);
  // plain copy bound for comparison
  {
    float* dst;
    CK(cudaMalloc(&dst, (size_t)S * pitch * 4 / 4));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaMemcpy(dst, y, (size_t)S * pitch, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(a));
    CK(cudaMemcpy(dst, y, (size_t)S * pitch, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-40s %8.3f ms  %7.1f GB/s (read+write)\n", "memcpy d2d (1/4 of y)", ms, 2.0 * S * pitch / ms / 1e6);
    CK(cudaFree(dst));
  }
  run<0, 256, 16, 8, 8, 1>("bulk TW256 GS16 ST8", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<0, 256, 32, 6, 8, 1>("bulk TW256 GS32 ST6", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<0, 128, 32, 8, 4, 1>("bulk TW128 GS32 ST8", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<0, 512, 16, 6, 8, 1>("bulk TW512 GS16 ST6", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<1, 256, 16, 8, 8, 2>("ldgsts TW256 GS16 ST8 P2", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<1, 256, 16, 8, 8, 4>("ldgsts TW256 GS16 ST8 P4", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<1, 128, 32, 8, 4, 4>("ldgsts TW128 GS32 ST8 P4", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<2, 256, 16, 8, 8, 1>("gather4 TW256 GS16 ST8", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<2, 256, 32, 6, 8, 1>("gather4 TW256 GS32 ST6", enc, y, pitch, T, d_order, S, out, sms, ref);
  run<2, 128, 32, 8, 4, 1>("gather4 TW128 GS32 ST8", enc, y, pitch, T, d_order, S, out, sms, ref);
  return 0;
}
