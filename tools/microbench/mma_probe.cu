// tcgen05.mma kind::f16 probe: canonical K-major SWIZZLE_NONE smem operands,
// fp32 accumulator in TMEM, split-fp16 (hi/lo) products for fp32-level accuracy.
//   D[m][n] = sum_k A[m][k] * B[n][k],  M = 128, N = 128, K = 128
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128, N = 128, K = 128;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// byte offset of element (r, k) of an R-row K-major canonical (no swizzle) operand
__device__ __forceinline__ int canon(int r, int k, int R) {
  return (k >> 4) * (R * 32) + (r >> 3) * 256 + ((k >> 3) & 1) * 128 + (r & 7) * 16 + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t sdesc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

template <int PRODUCTS, bool ATMEM>
__global__ void k_probe(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __half* Ah = (__half*)sm;                 // [M x K] hi
  __half* Al = (__half*)(sm + M * K * 2);   // lo
  __half* Bh = (__half*)(sm + 2 * M * K * 2);
  __half* Bl = (__half*)(sm + 2 * M * K * 2 + N * K * 2);
  __shared__ uint64_t bar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = A[i];
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *(__half*)((unsigned char*)Ah + canon(r, k, M)) = h;
    *(__half*)((unsigned char*)Al + canon(r, k, M)) = l;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i];
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *(__half*)((unsigned char*)Bh + canon(r, k, N)) = h;
    *(__half*)((unsigned char*)Bl + canon(r, k, N)) = l;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tbase;
  if (ATMEM) {  // row t of A -> TMEM lane t: column j = {A[t][2j], A[t][2j+1]} (hi at col 256, lo at 256 + K/2)
    const int t = tid;
    for (int part = 0; part < 2; ++part)
      for (int j0 = 0; j0 < K / 2; j0 += 8) {
        unsigned w[8];
        for (int j = 0; j < 8; ++j) {
          const float x0 = A[t * K + 2 * (j0 + j)], x1 = A[t * K + 2 * (j0 + j) + 1];
          const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
          const __half v0 = part ? __float2half_rn(x0 - __half2float(h0)) : h0;
          const __half v1 = part ? __float2half_rn(x1 - __half2float(h1)) : h1;
          w[j] = (unsigned)__half_as_ushort(v0) | ((unsigned)__half_as_ushort(v1) << 16);
        }
        const unsigned ta = tmem + ((unsigned)(32 * warp) << 16) + 256 + part * (K / 2) + j0;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]),
                     "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    const __half* As[3] = {Ah, Ah, Al};
    const __half* Bs[3] = {Bh, Bl, Bh};
    int first = 1;
    for (int p = 0; p < PRODUCTS; ++p)
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint64_t da = sdesc(su32(As[p]) + ks * M * 32);
        const uint64_t db = sdesc(su32(Bs[p]) + ks * N * 32);
        if (ATMEM) {
          const unsigned at = tmem + 256 + (p == 2 ? K / 2 : 0) + ks * 8;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(at), "l"(db), "r"(idesc), "r"(first ? 0 : 1));
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(first ? 0 : 1));
        }
        first = 0;
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
  }
  // wait for the MMA chain
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned ta = tmem + ((unsigned)(32 * warp) << 16);
  for (int c = 0; c < N; c += 16) {
    float v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                   "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                 : "r"(ta + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[(32 * warp + lane) * N + c + j] = v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  float *hA = (float*)malloc(M * K * 4), *hB = (float*)malloc(N * K * 4), *hD = (float*)malloc(M * N * 4);
  srand(1);
  auto rnd = [] { return (float)rand() / RAND_MAX * 2.f - 1.f; };
  for (int i = 0; i < M * K; ++i) hA[i] = rnd() * 3000.f;
  for (int i = 0; i < N * K; ++i) hB[i] = (rand() % 8 == 0) ? fabsf(rnd()) * 8000.f : 0.f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, M * K * 4)); CK(cudaMalloc(&dB, N * K * 4)); CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB, N * K * 4, cudaMemcpyHostToDevice));
  const int smem = 2 * M * K * 2 + 2 * N * K * 2;
  for (int prods : {1, 3, 4}) {
    if (prods == 1) { CK(cudaFuncSetAttribute(k_probe<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); k_probe<1, false><<<1, 128, smem>>>(dA, dB, dD); }
    else if (prods == 3) { CK(cudaFuncSetAttribute(k_probe<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); k_probe<3, false><<<1, 128, smem>>>(dA, dB, dD); }
    else { CK(cudaFuncSetAttribute(k_probe<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); k_probe<3, true><<<1, 128, smem>>>(dA, dB, dD); }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost));
    double num = 0, den = 0, maxe = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)hA[m * K + k] * hB[n * K + k];
        const double e = hD[m * N + n] - ref;
        num += e * e; den += ref * ref; maxe = fmax(maxe, fabs(e));
      }
    printf("variant=%d (4 = A from TMEM, 3 products)  rel L2 = %.3e  max abs err = %.3e  D[0][0]=%f\n", prods, sqrt(num / den), maxe, hD[0]);
  }
  return 0;
}
