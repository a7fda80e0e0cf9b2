// Tap-loop throughput probe, FFMA2 edition: pure FFMA vs FFMA2 issue, and the
// production pair loop (runtime-column TMEM loads) with packed FFMA2.
//  A) 4 warps/CTA x 4 CTAs/SM, 32x32b.x16, two directions interleaved (production k_render loop)
//  B) 24 warps/CTA x 1 CTA/SM, 16x64b.x16, one direction (2 threads per TMEM lane)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void ld32x32(float (&d)[16], unsigned ta) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
    : "=f"(d[0]),"=f"(d[1]),"=f"(d[2]),"=f"(d[3]),"=f"(d[4]),"=f"(d[5]),"=f"(d[6]),"=f"(d[7]),"=f"(d[8]),"=f"(d[9]),"=f"(d[10]),"=f"(d[11]),"=f"(d[12]),"=f"(d[13]),"=f"(d[14]),"=f"(d[15]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void ld16x64(float (&d)[16], unsigned ta) {
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
    : "=f"(d[0]),"=f"(d[1]),"=f"(d[2]),"=f"(d[3]),"=f"(d[4]),"=f"(d[5]),"=f"(d[6]),"=f"(d[7]),"=f"(d[8]),"=f"(d[9]),"=f"(d[10]),"=f"(d[11]),"=f"(d[12]),"=f"(d[13]),"=f"(d[14]),"=f"(d[15]) : "r"(ta) : "memory");
}
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float v) {
  asm("{\n\t.reg .b64 a, x, v;\n\tmov.b64 a, {%0,%1};\n\tmov.b64 x, {%2,%3};\n\tmov.b64 v, {%4,%4};\n\t"
      "fma.rn.f32x2 a, x, v, a;\n\tmov.b64 {%0,%1}, a;\n}" : "+f"(a0), "+f"(a1) : "f"(x0), "f"(x1), "f"(v));
}
template <bool PACKED>
__global__ void k_fma(float* out, float v, int iters) {
  float a[32];
  for (int i = 0; i < 32; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float x = v * 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if (PACKED) ffma2(a[i], a[i + 1], a[i], a[i + 1], x);
      else { a[i] = fmaf(a[i], x, v); a[i + 1] = fmaf(a[i + 1], x, v); }
    }
  }
  float t = 0; for (int i = 0; i < 32; ++i) t += a[i];
  if (t == 1234.5f) out[threadIdx.x] = t;
}
__device__ __forceinline__ void waitld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

constexpr int NNZ = 16;

template <int NW, int COLS, bool SHAPE16>
__global__ void k_taps(const int2* __restrict__ taps_g, int ndir, float* out, int iters) {
  __shared__ unsigned tb;
  __shared__ int2 s_taps[256 * NNZ];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&tb)), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < ndir * NNZ; i += blockDim.x) s_taps[i] = taps_g[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned tl;
  if (SHAPE16) {
    const int slot = warp >> 2;           // 0..5
    tl = tb + ((unsigned)(32 * (warp & 3) + 16 * (slot & 1)) << 16) + (slot >> 1) * 144;
  } else {
    tl = tb + ((unsigned)(32 * (warp & 3)) << 16) + (warp >> 2) * 128;
  }
  float tot = 0.f;
  for (int it = 0; it < iters; ++it) {
    if (!SHAPE16) {
      for (int d = 0; d < ndir; d += 2) {
        const int2* A = s_taps + d * NNZ;
        const int2* B = A + NNZ;
        float aA[16], aB[16], XA0[16], XB0[16], XA1[16], XB1[16];
        for (int r = 0; r < 16; ++r) { aA[r] = 0; aB[r] = 0; }
        int2 ta = A[0], tb2 = B[0];
        ld32x32(XA0, tl + ta.x); ld32x32(XB0, tl + tb2.x);
#pragma unroll
        for (int k = 0; k < NNZ; ++k) {
          const int2 na = A[k + 1 < NNZ ? k + 1 : k], nb = B[k + 1 < NNZ ? k + 1 : k];
          float(&XA)[16] = (k & 1) ? XA1 : XA0; float(&XB)[16] = (k & 1) ? XB1 : XB0;
          float(&YA)[16] = (k & 1) ? XA0 : XA1; float(&YB)[16] = (k & 1) ? XB0 : XB1;
          waitld();
          if (k + 1 < NNZ) { ld32x32(YA, tl + na.x); ld32x32(YB, tl + nb.x); }
          const float va = __int_as_float(ta.y), vb = __int_as_float(tb2.y);
#pragma unroll
          for (int r = 0; r < 16; r += 2) { ffma2(aA[r], aA[r + 1], XA[r], XA[r + 1], va); ffma2(aB[r], aB[r + 1], XB[r], XB[r + 1], vb); }
          ta = na; tb2 = nb;
        }
        for (int r = 0; r < 16; ++r) tot += aA[r] + aB[r];
      }
    } else {
      for (int d = 0; d < ndir; ++d) {
        const int2* A = s_taps + d * NNZ;
        float aA[16], X0[16], X1[16];
        for (int r = 0; r < 16; ++r) aA[r] = 0;
        int2 ta = A[0];
        ld16x64(X0, tl + ta.x);
#pragma unroll
        for (int k = 0; k < NNZ; ++k) {
          const int2 na = A[k + 1 < NNZ ? k + 1 : k];
          float(&X)[16] = (k & 1) ? X1 : X0; float(&Y)[16] = (k & 1) ? X0 : X1;
          waitld();
          if (k + 1 < NNZ) ld16x64(Y, tl + na.x);
          const float va = __int_as_float(ta.y);
#pragma unroll
          for (int r = 0; r < 16; ++r) aA[r] = fmaf(va, X[r], aA[r]);
          ta = na;
        }
        for (int r = 0; r < 16; ++r) tot += aA[r];
      }
    }
  }
  if (tot == 1234.5f) out[threadIdx.x] = tot;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "n"(COLS) : "memory");
}

int main() {
  const int ndir = 128, iters = 200;
  int2* h = (int2*)malloc(ndir * NNZ * 8);
  srand(3);
  for (int i = 0; i < ndir * NNZ; ++i) { float v = 0.5f; int vb; memcpy(&vb, &v, 4); h[i] = make_int2(rand() % 100, vb); }
  int2* d; CK(cudaMalloc(&d, ndir * NNZ * 8)); CK(cudaMemcpy(d, h, ndir * NNZ * 8, cudaMemcpyHostToDevice));
  float* o; CK(cudaMalloc(&o, 4096));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int ctas, int threads, double fma_per_thread_per_iter, const char* nm) {
    kern<<<ctas, threads>>>(d, ndir, o, 2); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); kern<<<ctas, threads>>>(d, ndir, o, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)ctas * threads * fma_per_thread_per_iter * iters;
    printf("%-40s %.3f ms  %.2f TFLOP/s  (%.1f%% of 74.4)\n", nm, ms, 2 * fma / (ms * 1e-3) / 1e12, 100 * 2 * fma / (ms * 1e-3) / 74.4e12);
  };
  {
    for (int pk = 0; pk < 2; ++pk) for (int wpsm : {16, 32, 64}) {
      auto kern = pk ? k_fma<true> : k_fma<false>;
      const int ctas = 148 * (wpsm / 8), threads = 256, it = 20000;
      kern<<<ctas, threads>>>(o, 1.0001f, 10); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0); kern<<<ctas, threads>>>(o, 1.0001f, it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * ctas * threads * 32.0 * it;
      printf("%s %2d warps/SM: %.2f TFLOP/s (%.1f%% of 74.4)\n", pk ? "FFMA2" : "FFMA ", wpsm, fl / (ms * 1e-3) / 1e12, 100 * fl / (ms * 1e-3) / 74.4e12);
    }
  }
  run(k_taps<4, 128, false>, 148 * 4, 128, (double)ndir * NNZ * 16, "A: 16 warps/SM, 32x32b pairs, FFMA2");
  run(k_taps<24, 512, true>, 148, 768, (double)ndir * NNZ * 16, "B: 24 warps/SM, 16x64b single");
  return 0;
}
