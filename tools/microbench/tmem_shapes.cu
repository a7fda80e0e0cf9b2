// Probe: which TMEM lane/column does each thread get for tcgen05.ld.16x64b / 16x128b / 16x256b?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  __shared__ unsigned tb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"((unsigned)__cvta_generic_to_shared(&tb)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned base = tb + ((unsigned)(32 * warp) << 16);
  // each thread writes value (lane_global*1000 + col) to its own lane row, cols 0..31
  int v[32];
  for (int c = 0; c < 32; ++c) v[c] = (32 * warp + lane) * 1000 + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
    :: "r"(base), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),
       "r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  int r[4];
  // 16x64b.x2: expect 2 regs per thread
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(base + 0) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (warp == 0) { out[lane * 4 + 0] = r[0]; out[lane * 4 + 1] = r[1]; }
  // 16x64b.x2 with lane offset 16
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(base + (16u << 16)) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (warp == 0) { out[128 + lane * 4 + 0] = r[0]; out[128 + lane * 4 + 1] = r[1]; }
  // 16x128b.x1: expect 2 regs
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(base + 0) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (warp == 0) { out[256 + lane * 4 + 0] = r[0]; out[256 + lane * 4 + 1] = r[1]; }
  // 16x256b.x1: expect 4 regs
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(base + 0) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (warp == 0) { for (int i = 0; i < 4; ++i) out[384 + lane * 4 + i] = r[i]; }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tb) : "memory");
}
int main() {
  int* d; cudaMalloc(&d, 512 * 4); cudaMemset(d, 0xff, 512 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err: %s\n", cudaGetErrorString(e));
  int h[512]; cudaMemcpy(h, d, 512 * 4, cudaMemcpyDeviceToHost);
  const char* names[4] = {"16x64b.x2", "16x64b.x2 lane+16", "16x128b.x1", "16x256b.x1"};
  for (int s = 0; s < 4; ++s) {
    printf("%s:\n", names[s]);
    for (int t = 0; t < 32; ++t) {
      printf(" t%02d:", t);
      for (int i = 0; i < (s == 3 ? 4 : 2); ++i) printf(" %6d", h[s * 128 + t * 4 + i]);
      if (t % 4 == 3) printf("\n");
    }
  }
  return 0;
}
