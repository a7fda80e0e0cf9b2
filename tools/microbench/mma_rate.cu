// tcgen05.mma kind::f16 issue-rate probe: cycles per MMA (M = 128, K = 16) for
// N in {64, 128, 256}, A from TMEM (TS) or shared memory (SS), B from shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
template <int N, bool TS>
__global__ void k_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<unsigned*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tm = tbase;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int ks = it & 7;
      const uint64_t db = sdesc(su32(sm) + 32768 + ks * N * 32 % 16384);
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tm), "r"(tm + 256 + 8 * ks), "l"(db), "r"(idesc), "r"(it > 0 ? 1 : 0));
      } else {
        const uint64_t da = sdesc(su32(sm) + ks * 4096);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(it > 0 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(su32(&bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int N, bool TS>
int run(long long* d, const char* nm) {
  const int smem = 64 * 1024, iters = 4096;
  CK(cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_rate<N, TS><<<148, 128, smem>>>(d, 64); CK(cudaDeviceSynchronize());
  k_rate<N, TS><<<148, 128, smem>>>(d, iters); CK(cudaDeviceSynchronize());
  long long h[148]; CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const double cyc = avg / iters, macs = 128.0 * N * 16;
  printf("%s N=%3d: %6.1f cycles/MMA  %6.0f MAC/cycle/SM  (%.0f%% of 4096)\n", nm, N, cyc, macs / cyc, 100 * macs / cyc / 4096);
  return 0;
}
int main() {
  long long* d; CK(cudaMalloc(&d, 148 * 8));
  run<64, true>(d, "TS"); run<128, true>(d, "TS"); run<256, true>(d, "TS");
  run<64, false>(d, "SS"); run<128, false>(d, "SS"); run<256, false>(d, "SS");
  return 0;
}
