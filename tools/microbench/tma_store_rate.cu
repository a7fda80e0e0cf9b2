// Store-throughput probe for the render epilogue's write pattern (cfg2:
// 2,500 rows x 441,199 fp32 = 4.41 GB).
//
// 1. k_store: every CTA (one per SM, W warps) walks 128-output x 128-direction
//    units as k_render_mma's epilogue does -- each warp stages 4 KB boxes in
//    shared memory and issues a 2-D TMA tensor store per box, two staging
//    buffers per warp -- by box shape ({32 t, 32 d} = the kernel's, {64, 16},
//    {128, 8}), row pitch (441,216 = 128-byte rows; 441,200 = 16-byte rows) and
//    unit order (blocked per CTA, or the kernel's groups of 6 CTAs on 6
//    consecutive tiles).
// 2. the same bytes through other paths: per-lane STG.32 (lane = t, the
//    tcgen05.ld layout), staged STG.128, contiguous 1-D bulk stores, a
//    contiguous STG.128 fill with values, cudaMemset of zeros.
// 3. TMA and STG.128 boxes mixed in one kernel.
//
// Findings (profiles/r2_store_ceiling.txt): cudaMemset of zeros (7.27 TB/s) is
// not a ceiling for data -- non-zero contiguous stores top out at 6.2-6.45
// TB/s, the epilogue's row pattern at 5.9-6.4 TB/s with >= 256-byte box rows
// and 128-byte-aligned rows; 128-byte box rows cost ~15%.
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
                                                  int units_per_cta, int inter) {
  extern __shared__ __align__(128) float st[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* mine = st + warp * 2 * (BT * BD);
  constexpr int BOXES = (128 / BT) * (128 / BD);  // per unit
  int sbuf = 0;
  const long long u0 = (long long)blockIdx.x * units_per_cta;
  for (long long i = 0; i < units_per_cta; ++i) {
    // blocked: CTA b walks units [b*per, (b+1)*per), tile fastest; interleaved:
    // unit i*grid + b with the chunk fastest inside a tile group of the grid
    long long u = inter ? i * gridDim.x + blockIdx.x : u0 + i;
    int tile, chunk;
    if (inter == 3) {  // k_render_mma's order: groups of 6 CTAs on 6 consecutive tiles, chunk fastest
      const long long cl = blockIdx.x / 6, cr = blockIdx.x % 6, ncl = gridDim.x / 6;
      const long long groups = ((long long)n_tiles + 5) / 6;
      const long long g0 = groups * cl / ncl, g1 = groups * (cl + 1) / ncl;
      const long long gu = g0 * n_chunks + i;
      if (blockIdx.x >= ncl * 6 || gu >= g1 * n_chunks) break;
      chunk = (int)(gu % n_chunks);
      tile = (int)((gu / n_chunks) * 6 + cr);
      if (tile >= n_tiles) continue;
    } else if (inter == 2) {  // all CTAs on one chunk, adjacent tiles
      const long long grp = u / ((long long)gridDim.x * n_chunks), r = u % ((long long)gridDim.x * n_chunks);
      chunk = (int)(r / gridDim.x);
      tile = (int)(grp * gridDim.x + r % gridDim.x);
      if (tile >= n_tiles) continue;
    } else {
      tile = (int)(u % n_tiles);
      chunk = (int)((u / n_tiles) % n_chunks);
    }
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
static int run(EncodeTiledFn enc, float* out, long long rows, long long len, long long pitch, int sms, int warps,
               int inter = 0) {
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
  kern<<<sms, warps * 32, smem>>>(tm, n_tiles, n_chunks, inter == 2 ? per + n_chunks : inter == 3 ? 2 * per + 2 * n_chunks : per, inter);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<sms, warps * 32, smem>>>(tm, n_tiles, n_chunks, inter == 2 ? per + n_chunks : inter == 3 ? 2 * per + 2 * n_chunks : per, inter);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)rows * len * 4;
  printf("box {%3d t, %2d d}  %s  %2d warps  pitch %lld  order %s  %.3f ms  %.0f GB/s\n", BT, BD,
         STS ? "STS+TMA" : "TMA only", warps, pitch, inter == 0 ? "blocked" : inter == 1 ? "strided" : inter == 2 ? "chunk-sync" : "6-cta groups",
         best, bytes / best / 1e6);
  return 0;
}

// direct stores: lane = t (the tcgen05.ld 32x32b row), one 128-byte row
// segment per instruction, no staging (CS: st.global.cs)
template <int CS>
__global__ void __launch_bounds__(512, 1) k_stg(float* out, long long pitch, int len, int rows, int n_tiles,
                                                int n_chunks, int units_per_cta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (long long i = 0; i < units_per_cta; ++i) {
    const long long u = (long long)blockIdx.x * units_per_cta + i;
    const int tile = (int)(u % n_tiles), chunk = (int)((u / n_tiles) % n_chunks);
    for (int b = warp; b < 16; b += nw) {  // 4 lane quarters x 4 column blocks of 32
      const int q = b & 3, cb = b >> 2;
      const int t = tile * 128 + 32 * q + lane;
      const int d0 = chunk * 128 + 32 * cb;
      if (t >= len) continue;
      float* p = out + (long long)d0 * pitch + t;
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        if (d0 + j < rows) {
          const float v = (float)(j + u);
          if (CS) asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p + (long long)j * pitch), "f"(v) : "memory");
          else p[(long long)j * pitch] = v;
        }
      }
    }
  }
}

template <int CS>
static int run_stg(float* out, long long rows, long long len, long long pitch, int sms, int warps) {
  const int n_tiles = (int)((len + 127) / 128), n_chunks = (int)((rows + 127) / 128);
  const long long units = (long long)n_tiles * n_chunks;
  const int per = (int)((units + sms - 1) / sms);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_stg<CS><<<sms, warps * 32>>>(out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_stg<CS><<<sms, warps * 32>>>(out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("direct STG%s lane = t  %2d warps  pitch %lld  %.3f ms  %.0f GB/s\n", CS ? ".cs" : "", warps, pitch, best,
         (double)rows * len * 4 / best / 1e6);
  return 0;
}

// staged vector stores: STS [d][t] as the TMA path, then LDS.128 + STG.128
// (lane = 4 consecutive t of one row; a warp instruction = 4 rows x 128 B)
template <int CS>
__global__ void __launch_bounds__(512, 1) k_stg4(float* out, long long pitch, int len, int rows, int n_tiles,
                                                 int n_chunks, int units_per_cta) {
  extern __shared__ __align__(128) float st[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* buf = st + warp * 32 * 33;
  for (long long i = 0; i < units_per_cta; ++i) {
    const long long u = (long long)blockIdx.x * units_per_cta + i;
    const int tile = (int)(u % n_tiles), chunk = (int)((u / n_tiles) % n_chunks);
    for (int b = warp; b < 16; b += nw) {
      const int q = b & 3, cb = b >> 2;
      const int t0 = tile * 128 + 32 * q;
      const int d0 = chunk * 128 + 32 * cb;
#pragma unroll
      for (int j = 0; j < 32; ++j) buf[j * 32 + lane] = (float)(j + u);
      __syncwarp();
      const int rr = lane >> 3, tt = 4 * (lane & 7);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int d = 4 * k + rr;
        const float4 v = *reinterpret_cast<const float4*>(buf + d * 32 + tt);
        if (d0 + d < rows && t0 + tt < len) {
          float* p = out + (long long)(d0 + d) * pitch + t0 + tt;
          if (CS) asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
          else *reinterpret_cast<float4*>(p) = v;
        }
      }
      __syncwarp();
    }
  }
}

template <int CS>
static int run_stg4(float* out, long long rows, long long len, long long pitch, int sms, int warps) {
  const int n_tiles = (int)((len + 127) / 128), n_chunks = (int)((rows + 127) / 128);
  const long long units = (long long)n_tiles * n_chunks;
  const int per = (int)((units + sms - 1) / sms);
  const int smem = warps * 32 * 33 * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_stg4<CS><<<sms, warps * 32, smem>>>(out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_stg4<CS><<<sms, warps * 32, smem>>>(out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("staged STG.128%s  %2d warps  pitch %lld  %.3f ms  %.0f GB/s\n", CS ? ".cs" : "", warps, pitch, best,
         (double)rows * len * 4 / best / 1e6);
  return 0;
}

// contiguous bulk stores (cp.async.bulk.global.shared, 1-D): box-sized pieces of
// one linear buffer, to separate the TMA store path from the row pattern
template <int BYTES>
__global__ void __launch_bounds__(512, 1) k_bulk1d(float* out, long long total_pieces, int per) {
  extern __shared__ __align__(128) float st[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int NF = BYTES / 4;
  float* mine = st + warp * 2 * NF;
  int sbuf = 0;
  for (int i = warp; i < per; i += nw) {
    const long long pc = (long long)blockIdx.x * per + i;
    if (pc >= total_pieces) break;
    float* buf = mine + sbuf * NF;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
    for (int k = lane; k < NF; k += 32) buf[k] = (float)(k + i);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + pc * NF),
                   "r"(su32(buf)), "r"(BYTES) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    sbuf ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int BYTES>
static int run_bulk1d(float* out, long long floats, int sms, int warps) {
  const long long pieces = floats * 4 / BYTES;
  const int per = (int)((pieces + sms - 1) / sms);
  const int smem = warps * 2 * BYTES;
  CK(cudaFuncSetAttribute(k_bulk1d<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_bulk1d<BYTES><<<sms, warps * 32, smem>>>(out, pieces, per);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_bulk1d<BYTES><<<sms, warps * 32, smem>>>(out, pieces, per);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("contiguous bulk store %5d B  %2d warps  %.3f ms  %.0f GB/s\n", BYTES, warps, best,
         (double)pieces * BYTES / best / 1e6);
  return 0;
}

// plain vector stores: contiguous grid-stride fill with values, and the unit
// pattern with one 512-byte row segment (128 t) per warp instruction
__global__ void __launch_bounds__(512) k_fill4(float4* out, long long n4) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    out[i] = make_float4((float)i, 1.f, 2.f, 3.f);
}

__global__ void __launch_bounds__(512, 1) k_row4(float* out, long long pitch, int len, int rows, int n_tiles,
                                                 int n_chunks, int units_per_cta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (long long i = 0; i < units_per_cta; ++i) {
    const long long u = (long long)blockIdx.x * units_per_cta + i;
    const int tile = (int)(u % n_tiles), chunk = (int)((u / n_tiles) % n_chunks);
    const int t = tile * 128 + 4 * lane;
    for (int r = warp; r < 128; r += nw) {
      const int d = chunk * 128 + r;
      if (d < rows && t < len)
        *reinterpret_cast<float4*>(out + (long long)d * pitch + t) = make_float4((float)r, 1.f, 2.f, (float)u);
    }
  }
}

static int run_plain(float* out, long long rows, long long len, long long pitch, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n_tiles = (int)((len + 127) / 128), n_chunks = (int)((rows + 127) / 128);
  const long long units = (long long)n_tiles * n_chunks;
  const int per = (int)((units + sms - 1) / sms);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(a);
      if (mode == 0) k_fill4<<<sms * 4, 512>>>(reinterpret_cast<float4*>(out), rows * pitch / 4);
      else k_row4<<<sms, mode == 1 ? 256 : 512>>>(out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (r && ms < best) best = ms;
    }
    printf("%s pitch %lld  %.3f ms  %.0f GB/s\n", mode == 0 ? "contiguous STG.128 fill" : mode == 1 ? "row STG.128 8 warps" : "row STG.128 16 warps",
           pitch, best, (double)(mode == 0 ? rows * pitch : rows * len) * 4 / best / 1e6);
  }
  return 0;
}

// half the boxes through TMA ({64 t, 16 d}), half through staged STG.128 by
// the same warps: do the two store paths have separate per-SM limits?
__global__ void __launch_bounds__(512, 1) k_mixed(const __grid_constant__ CUtensorMap tm, float* out, long long pitch,
                                                  int len, int rows, int n_tiles, int n_chunks, int units_per_cta,
                                                  int stg_every) {
  extern __shared__ __align__(128) float st[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* mine = st + warp * 3 * 1024;
  int sbuf = 0;
  for (long long i = 0; i < units_per_cta; ++i) {
    const long long u = (long long)blockIdx.x * units_per_cta + i;
    const int tile = (int)(u % n_tiles), chunk = (int)((u / n_tiles) % n_chunks);
    for (int b = warp; b < 16; b += nw) {  // 16 boxes of {64 t, 16 d} per unit
      const int bt = b & 1, bd = b >> 1;
      const int t0 = tile * 128 + 64 * bt, d0 = chunk * 128 + 16 * bd;
      if (stg_every && (b % stg_every) == stg_every - 1) {
        float* buf = mine + 2048;
        for (int j = lane; j < 1024; j += 32) buf[j] = (float)(j + u);
        __syncwarp();
        // lane -> row (lane >> 4) + 2k, t = 4 * (lane & 15): 2 rows x 256 B per instruction
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int d = 2 * k + (lane >> 4), tt = 4 * (lane & 15);
          const float4 v = *reinterpret_cast<const float4*>(buf + d * 64 + tt);
          if (d0 + d < rows && t0 + tt < len) *reinterpret_cast<float4*>(out + (long long)(d0 + d) * pitch + t0 + tt) = v;
        }
        __syncwarp();
      } else {
        float* buf = mine + sbuf * 1024;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        for (int j = lane; j < 1024; j += 32) buf[j] = (float)(j + u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm),
                       "r"(su32(buf)), "r"(t0), "r"(d0) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        sbuf ^= 1;
      }
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int run_mixed(EncodeTiledFn enc, float* out, long long rows, long long len, long long pitch, int sms, int warps,
                     int stg_every) {
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)len, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  const cuuint32_t box[2] = {64, 16};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 1;
  const int n_tiles = (int)((len + 127) / 128), n_chunks = (int)((rows + 127) / 128);
  const long long units = (long long)n_tiles * n_chunks;
  const int per = (int)((units + sms - 1) / sms);
  const int smem = warps * 3 * 4096;
  CK(cudaFuncSetAttribute(k_mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    k_mixed<<<sms, warps * 32, smem>>>(tm, out, pitch, (int)len, (int)rows, n_tiles, n_chunks, per, stg_every);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  printf("mixed TMA {64,16} + STG.128, every %d-th box by STG  %2d warps  %.3f ms  %.0f GB/s\n", stg_every, warps, best,
         (double)rows * len * 4 / best / 1e6);
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
  // 1. the render epilogue's pattern: box shape x row pitch x unit order
  for (long long pp : {pitch, 441200ll})  // 128-byte rows / 16-byte rows
    for (int inter : {0, 3}) {
      run<32, 32, true>(enc, out, rows, len, pp, sms, 8, inter);
      run<64, 16, true>(enc, out, rows, len, pp, sms, 8, inter);
      run<128, 8, true>(enc, out, rows, len, pp, sms, 8, inter);
    }
  // 2. other store paths for the same bytes
  for (int w : {8, 16}) {
    run_stg<0>(out, rows, len, pitch, sms, w);
    run_stg4<0>(out, rows, len, pitch, sms, 8);
  }
  run_bulk1d<4096>(out, rows * pitch, sms, 8);
  run_plain(out, rows, len, pitch, sms);
  // 3. TMA and LSU stores together
  for (int ev : {0, 4, 2}) run_mixed(enc, out, rows, len, pitch, sms, 8, ev);
  // plain fill for the ceiling
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    cudaMemsetAsync(out, 0, rows * pitch * 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  printf("cudaMemset (zeros) %.3f ms  %.0f GB/s\n", best, rows * pitch * 4.0 / best / 1e6);
  cudaFree(out);
  return 0;
}
