// TMEM -> register load throughput probe (design microbenchmark, not product code)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

template <int NW, int COLS, int MODE>
__global__ __launch_bounds__(NW * 32) void k_bw(float* out, int iters) {
  __shared__ unsigned tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&tb)), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned base = tb + ((unsigned)(32 * (warp & 3)) << 16) + (warp >> 2) * (COLS / (NW / 4));
  float s = 0.f, a[16];
  for (int i = 0; i < 16; ++i) a[i] = 0.f;
  float v = out[threadIdx.x & 7];
  for (int it = 0; it < iters; ++it) {
    unsigned ta = base + ((it * 7) & 63);
    float r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(r[0]),"=f"(r[1]),"=f"(r[2]),"=f"(r[3]),"=f"(r[4]),"=f"(r[5]),"=f"(r[6]),"=f"(r[7]),
        "=f"(r[8]),"=f"(r[9]),"=f"(r[10]),"=f"(r[11]),"=f"(r[12]),"=f"(r[13]),"=f"(r[14]),"=f"(r[15]) : "r"(ta) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (MODE == 0) { s += r[it & 15]; }
    else {
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] = fmaf(v, r[j], a[j]);
    }
  }
  for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "n"(COLS) : "memory");
}

int main() {
  float* d; CK(cudaMalloc(&d, 148 * 8 * 512 * 4)); CK(cudaMemset(d, 0, 148 * 8 * 512 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  auto run = [&](auto kern, int nw, int ctas_per_sm, const char* nm) {
    int grid = 148 * ctas_per_sm;
    kern<<<grid, nw * 32>>>(d, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); kern<<<grid, nw * 32>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double bytes = (double)grid * nw * 32 * 16 * 4 * iters;
    printf("%-34s %s %.3f ms  %.1f B/clk/SM @1.965GHz  FMA %.1f TF\n", nm, cudaGetErrorString(err), ms,
           bytes / (ms * 1e-3) / 148 / 1.965e9, 2.0 * grid * nw * 32 * 16.0 * iters / (ms * 1e-3) / 1e12);
  };
  run(k_bw<4, 128, 0>, 4, 4, "ld only 4w x4cta (16w/SM)");
  run(k_bw<4, 128, 1>, 4, 4, "ld+16fma 4w x4cta (16w/SM)");
  run(k_bw<8, 256, 0>, 8, 2, "ld only 8w x2cta (16w/SM)");
  run(k_bw<8, 256, 1>, 8, 2, "ld+16fma 8w x2cta");
  run(k_bw<4, 256, 1>, 4, 2, "ld+16fma 4w x2cta (8w/SM)");
  run(k_bw<16, 512, 1>, 16, 1, "ld+16fma 16w x1cta (16w/SM)");
  return 0;
}
