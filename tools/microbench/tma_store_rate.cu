// TMA tensor-store throughput probe for the render epilogue's write pattern.
//
// Output: rows x pitch fp32 (2,500 x 441,216 = 4.41 GB, the cfg2 shape).  Every
// CTA (one per SM, W warps) walks 128-output x 128-direction units exactly as
// k_render_mma's epilogue does -- each warp owns 4 KB boxes of the unit,
// stages them in shared memory (STS, or nothing with --nosts) and issues a
// 3-D TMA tensor store per box, two staging buffers per warp -- so the
// measured rate is the store path alone (no MMA, no TMEM, no G traffic).
// Box shapes: {32 t, 32 d} (the kernel's), {64, 16}, {128, 8}, {256, 4}.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_store_rate tma_store_rate.cu -lcuda
//   ./tma_store_rate
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e = (x);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                   \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// unit = (tile of 128 t, chunk of 128 d); a warp stores boxes bt x bd covering
// its share of the unit's 128 x 128 outputs; W warps split the unit's boxes
template <int BT, int BD, bool STS>
__global__ void __launch_bounds__(512, 1) k_store(const __grid_constant__ CUtensorMap tm, int n_tiles, int n_chunks,
                                                  int units_per_cta) {
  extern __shared__ __align__(128) float st[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* mine = st + warp * 2 * (BT * BD);
  constexpr int BOXES = (128 / BT) * (128 / BD);  // per unit
  int sbuf = 0;
  const long long u0 = (long long)blockIdx.x * units_per_cta;
  for (long long u = u0; u < u0 + units_per_cta; ++u) {
    const int tile = (int)(u % n_tiles), chunk = (int)((u / n_tiles) % n_chunks);
    for (int b = warp; b < BOXES; b += nw) {
      const int bt = b % (128 / BT), bd = b / (128 / BT);
      float* buf = mine + sbuf * BT * BD;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      if (STS) {
        for (int i = lane; i < BT * BD; i += 32) buf[i] = (float)(i + u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
      }
      if (lane == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                     "r"(su32(buf)), "r"(tile * 128 + bt * BT), "r"(chunk * 128 + bd * BD)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      sbuf ^= 1;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int BT, int BD, bool STS>
static int run(EncodeTiledFn enc, float* out, long long rows, long long len, long long pitch, int sms, int warps) {
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)len, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  const cuuint32_t box[2] = {BT, BD};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int n_tiles = (int)((len + 127) / 128), n_chunks = (int)((rows + 127) / 128);
  const long long units = (long long)n_tiles * n_chunks;
  const int per = (int)((units + sms - 1) / sms);
  const int smem = warps * 2 * BT * BD * 4;
  auto kern = k_store<BT, BD, STS>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<sms, warps * 32, smem>>>(tm, n_tiles, n_chunks, per);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<sms, warps * 32, smem>>>(tm, n_tiles, n_chunks, per);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)rows * len * 4;
  printf("box {%3d t, %2d d}  %s  %2d warps  %.3f ms  %.0f GB/s\n", BT, BD, STS ? "STS+TMA" : "TMA only", warps,
         best, bytes / best / 1e6);
  return 0;
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return 1;
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long rows = 2500, len = 441199, pitch = 441216;
  float* out = nullptr;
  CK(cudaMalloc(&out, rows * pitch * 4));
  for (int w : {8, 16}) {
    run<32, 32, true>(enc, out, rows, len, pitch, sms, w);
    run<32, 32, false>(enc, out, rows, len, pitch, sms, w);
    run<64, 16, true>(enc, out, rows, len, pitch, sms, w);
    run<128, 8, true>(enc, out, rows, len, pitch, sms, w);
    run<256, 4, true>(enc, out, rows, len, pitch, sms, w);
  }
  cudaFree(out);
  return 0;
}
