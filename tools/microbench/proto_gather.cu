// Design microbenchmark (not product code): compares ways to apply a sparse
// per-direction tap list to a shared resonance-filtered signal on sm_100a.
//   A) register window + warp-uniform jump table (one case per tap offset)
//   B) shared-memory gather, one LDS per FMA (baseline)
//   C) FFMA throughput probe
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o proto proto_gather.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cstring>
static int f2i(float f){int i; memcpy(&i,&f,4); return i;}
static float i2f(int i){float f; memcpy(&f,&i,4); return f;}
#include <cuda_runtime.h>
#include "jt_asm.inc"
#include "jt_asm2.inc"
#include "static_asm.inc"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int O, int R, int KW, int N>
__device__ __forceinline__ void tap_fma(float (&acc)[R], const float (&win)[N], float v) {
  if constexpr (O < KW) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = fmaf(v, win[r + KW - O], acc[r]);
  }
}

#define JC1(o) case (o): tap_fma<(o), R, KW, R + KW>(acc, win, v); break;
#define JC4(o) JC1(o) JC1(o + 1) JC1(o + 2) JC1(o + 3)
#define JC16(o) JC4(o) JC4(o + 4) JC4(o + 8) JC4(o + 12)
#define JC64(o) JC16(o) JC16(o + 16) JC16(o + 32) JC16(o + 48)

template <int R, int KW, int MINB>
__global__ __launch_bounds__(128, MINB) void k_jumptable(const float* __restrict__ yf, int nyf,
                                                          const int2* __restrict__ taps, int nnz,
                                                          int dirs_per_cta, float* __restrict__ out,
                                                          int out_len, long pitch) {
  constexpr int W = 128 * R;
  __shared__ __align__(16) float s[W + KW];
  const int T0 = blockIdx.x * W;
  for (int i = threadIdx.x; i < W + KW; i += 128) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tl = warp * 32 * R + lane * R;
  float win[R + KW];
#pragma unroll
  for (int i = 0; i < (R + KW) / 4; ++i) {
    float4 q = *reinterpret_cast<const float4*>(&s[tl + 4 * i]);
    win[4 * i] = q.x; win[4 * i + 1] = q.y; win[4 * i + 2] = q.z; win[4 * i + 3] = q.w;
  }
  const int d0 = blockIdx.y * dirs_per_cta;
  for (int d = d0; d < d0 + dirs_per_cta; ++d) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const int2* tp = taps + (long)d * nnz;
    for (int k = 0; k < nnz; ++k) {
      int2 tv = tp[k];
      const float v = __int_as_float(tv.y);
      switch (tv.x) {
        JC64(0) JC16(64) JC16(80) JC4(96)
        default: __builtin_unreachable();
      }
    }
    float* o = out + d * pitch + T0 + tl;
    if (T0 + tl + R <= out_len) {
#pragma unroll
      for (int r = 0; r < R; r += 4)
        __stcs(reinterpret_cast<float4*>(o + r), make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) if (T0 + tl + r < out_len) o[r] = acc[r];
    }
  }
}


#define JT_ASM(R, KW) JT_ASM_R##R##_K##KW
template <int R, int KW, int MINB> struct JtAsm;
#define DEF_JT(R_, KW_) template <int MINB> struct JtAsm<R_, KW_, MINB> { \
  static __device__ __forceinline__ void run(float (&acc)[R_], const float (&win)[R_ + KW_], const int2* p) { \
    asm volatile(JT_ASM_R##R_##_K##KW_ : JT_OUTS_R##R_ : JT_INS_R##R_##_K##KW_, "l"(p) : "memory"); } };
DEF_JT(20, 100)
DEF_JT(12, 100)
DEF_JT(28, 100)

template <int R, int KW, int MINB>
__global__ __launch_bounds__(128, MINB) void k_jtasm(const float* __restrict__ yf, int nyf,
                                                          const int2* __restrict__ taps, int stride,
                                                          int dirs_per_cta, float* __restrict__ out,
                                                          int out_len, long pitch) {
  constexpr int W = 128 * R;
  __shared__ __align__(16) float s[W + KW];
  const int T0 = blockIdx.x * W;
  for (int i = threadIdx.x; i < W + KW; i += 128) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tl = warp * 32 * R + lane * R;
  float win[R + KW];
#pragma unroll
  for (int i = 0; i < (R + KW) / 4; ++i) {
    float4 q = *reinterpret_cast<const float4*>(&s[tl + 4 * i]);
    win[4 * i] = q.x; win[4 * i + 1] = q.y; win[4 * i + 2] = q.z; win[4 * i + 3] = q.w;
  }
  const int d0 = blockIdx.y * dirs_per_cta;
  for (int d = d0; d < d0 + dirs_per_cta; ++d) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    JtAsm<R, KW, MINB>::run(acc, win, taps + (long)d * stride);
    float* o = out + d * pitch + T0 + tl;
    if (T0 + tl + R <= out_len) {
#pragma unroll
      for (int r = 0; r < R; r += 4)
        __stcs(reinterpret_cast<float4*>(o + r), make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) if (T0 + tl + r < out_len) o[r] = acc[r];
    }
  }
}


template <int R, int KW> struct JtAsm2;
#define DEF_JT2(R_, KW_) template <> struct JtAsm2<R_, KW_> { \
  static __device__ __forceinline__ void run(float (&acc)[R_], const float (&win)[R_ + KW_], unsigned p) { \
    asm volatile(JT2_ASM_R##R_##_K##KW_ : JT_OUTS2_R##R_ : JT_INS2_R##R_##_K##KW_, "r"(p) : "memory"); } };
DEF_JT2(20, 100)
DEF_JT2(20, 52)
DEF_JT2(36, 52)
DEF_JT2(12, 52)
DEF_JT2(12, 100)
DEF_JT2(28, 100)
__device__ __forceinline__ void bulk_store2(float* gdst, const float* ssrc, int bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int R, int MINB, int KW>
__global__ __launch_bounds__(128, MINB) void k_jtasm2(const float* __restrict__ yf, int nyf,
                                                          const int2* __restrict__ taps, int stride,
                                                          int dirs_per_cta, float* __restrict__ out,
                                                          int out_len, long pitch) {
  constexpr int W = 128 * R;
  extern __shared__ __align__(128) float s[];
  float* stage = s + W + KW + 28 + (threadIdx.x >> 5) * 3 * 32 * R;  // 3 slots per warp
  int2* stp = reinterpret_cast<int2*>(s + W + KW + 28 + 4 * 3 * 32 * R);
  const int T0 = blockIdx.x * W;
  const int d0 = blockIdx.y * dirs_per_cta;
  for (int i = threadIdx.x; i < W + KW; i += 128) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  for (int i = threadIdx.x; i < dirs_per_cta * stride; i += 128) stp[i] = taps[(long)d0 * stride + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tl = warp * 32 * R + lane * R;
  float win[R + KW];
#pragma unroll
  for (int i = 0; i < (R + KW) / 4; ++i) {
    float4 q = *reinterpret_cast<const float4*>(&s[tl + 4 * i]);
    win[4 * i] = q.x; win[4 * i + 1] = q.y; win[4 * i + 2] = q.z; win[4 * i + 3] = q.w;
  }
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(stp);
  const bool full = (T0 + warp * 32 * R + 32 * R <= out_len);
  int slot = 0;
  for (int dd = 0; dd < dirs_per_cta; ++dd) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    JtAsm2<R, KW>::run(acc, win, sbase + dd * stride * 8);
    float* st = stage + slot * 32 * R;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; r += 4)
      *reinterpret_cast<float4*>(st + lane * R + r) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
    __syncwarp();
    float* o = out + (d0 + dd) * pitch + T0 + warp * 32 * R;
    if (full) {
      if (lane == 0) bulk_store2(o, st, 32 * R * 4);
    } else {
      for (int i = lane; i < 32 * R; i += 32) if (T0 + warp * 32 * R + i < out_len) o[i] = st[i];
    }
    slot = (slot == 2) ? 0 : slot + 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// E) TMEM-resident window: dynamic column index per tap, no control flow
template <int N> struct TLd;
template <> struct TLd<16> {
  static __device__ __forceinline__ void ld(float (&d)[16], unsigned ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(d[0]),"=f"(d[1]),"=f"(d[2]),"=f"(d[3]),"=f"(d[4]),"=f"(d[5]),"=f"(d[6]),"=f"(d[7]),
        "=f"(d[8]),"=f"(d[9]),"=f"(d[10]),"=f"(d[11]),"=f"(d[12]),"=f"(d[13]),"=f"(d[14]),"=f"(d[15]) : "r"(ta) : "memory");
  }
  static __device__ __forceinline__ void st(const float (&d)[16], unsigned ta) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :: "r"(ta), "f"(d[0]),"f"(d[1]),"f"(d[2]),"f"(d[3]),"f"(d[4]),"f"(d[5]),"f"(d[6]),"f"(d[7]),
        "f"(d[8]),"f"(d[9]),"f"(d[10]),"f"(d[11]),"f"(d[12]),"f"(d[13]),"f"(d[14]),"f"(d[15]) : "memory");
  }
};
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// R = 16 * RB outputs per lane; window = R + KW columns; NW warps; COLS allocated per CTA
template <int RB, int NW, int COLS, int MINB>
__global__ __launch_bounds__(NW * 32, MINB) void k_tmem(const float* __restrict__ yf, int nyf,
                                                       const int2* __restrict__ taps, int stride,
                                                       int dirs_per_cta, float* __restrict__ out,
                                                       int out_len, long pitch) {
  constexpr int R = 16 * RB, KW = 100, W = NW * 32 * R;
  constexpr int WC = ((R + KW + 15) / 16) * 16;  // window columns per warp
  static_assert(WC * (NW / 4) <= COLS, "tmem");
  extern __shared__ __align__(128) float s[];
  __shared__ unsigned tbase_s;
  float* stage_base = s + W + KW + 28;
  int2* stp = reinterpret_cast<int2*>(stage_base + NW * 3 * 32 * R);
  const int T0 = blockIdx.x * W;
  const int d0 = blockIdx.y * dirs_per_cta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&tbase_s)), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < W + KW; i += NW * 32) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  for (int i = threadIdx.x; i < dirs_per_cta * stride; i += NW * 32) {
    int2 tv = taps[(long)d0 * stride + i];
    stp[i] = make_int2(KW - tv.x, tv.y);  // window column of the tap
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = tbase_s + ((unsigned)(32 * (warp & 3)) << 16) + (warp >> 2) * WC;
  const int tl = warp * 32 * R + lane * R;
  // write this lane's window into its TMEM row
#pragma unroll
  for (int c = 0; c < WC; c += 16) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      float4 q = (c + i < R + KW) ? *reinterpret_cast<const float4*>(&s[tl + c + i]) : make_float4(0, 0, 0, 0);
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
    TLd<16>::st(v, tbase + c);
  }
  tmem_wait_st();
  float* stage = stage_base + warp * 3 * 32 * R;
  const bool full = (T0 + warp * 32 * R + 32 * R <= out_len);
  int slot = 0;
  for (int dd = 0; dd < dirs_per_cta; ++dd) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const int2* tp = stp + dd * stride;
    int2 cur = tp[0];
    float bufA[R], bufB[R];
#pragma unroll
    for (int b = 0; b < RB; ++b) TLd<16>::ld(*reinterpret_cast<float(*)[16]>(&bufA[16 * b]), tbase + cur.x + 16 * b);
    int k = 0;
    const int nnz = stride - 1;
    while (true) {
      tmem_wait_ld();
      int2 nxt = tp[k + 1];
      if (k + 1 < nnz) {
#pragma unroll
        for (int b = 0; b < RB; ++b) TLd<16>::ld(*reinterpret_cast<float(*)[16]>(&bufB[16 * b]), tbase + nxt.x + 16 * b);
      }
      const float v = __int_as_float(cur.y);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fmaf(v, bufA[r], acc[r]);
      if (++k >= nnz) break;
      cur = nxt;
      tmem_wait_ld();
      nxt = tp[k + 1];
      if (k + 1 < nnz) {
#pragma unroll
        for (int b = 0; b < RB; ++b) TLd<16>::ld(*reinterpret_cast<float(*)[16]>(&bufA[16 * b]), tbase + nxt.x + 16 * b);
      }
      const float v2 = __int_as_float(cur.y);
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = fmaf(v2, bufB[r], acc[r]);
      if (++k >= nnz) break;
      cur = nxt;
    }
    float* st = stage + slot * 32 * R;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; r += 4)
      *reinterpret_cast<float4*>(st + lane * R + r) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
    __syncwarp();
    float* o = out + (d0 + dd) * pitch + T0 + warp * 32 * R;
    if (full) {
      if (lane == 0) bulk_store2(o, st, 32 * R * 4);
    } else {
      for (int i = lane; i < 32 * R; i += 32) if (T0 + warp * 32 * R + i < out_len) o[i] = st[i];
    }
    slot = (slot == 2) ? 0 : slot + 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase_s), "n"(COLS) : "memory");
}


template <> struct TLd<32> {
  static __device__ __forceinline__ void ld(float (&d)[32], unsigned ta) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=f"(d[0]),"=f"(d[1]),"=f"(d[2]),"=f"(d[3]),"=f"(d[4]),"=f"(d[5]),"=f"(d[6]),"=f"(d[7]),
        "=f"(d[8]),"=f"(d[9]),"=f"(d[10]),"=f"(d[11]),"=f"(d[12]),"=f"(d[13]),"=f"(d[14]),"=f"(d[15]),
        "=f"(d[16]),"=f"(d[17]),"=f"(d[18]),"=f"(d[19]),"=f"(d[20]),"=f"(d[21]),"=f"(d[22]),"=f"(d[23]),
        "=f"(d[24]),"=f"(d[25]),"=f"(d[26]),"=f"(d[27]),"=f"(d[28]),"=f"(d[29]),"=f"(d[30]),"=f"(d[31]) : "r"(ta) : "memory");
  }
};
// F) TMEM window, pipelined, fully unrolled fixed-NNZ tap loop, taps (col, v) in smem
template <int R, int NW, int COLS, int MINB, int NNZ>
__global__ __launch_bounds__(NW * 32, MINB) void k_tmem2(const float* __restrict__ yf, int nyf,
                                                       const int2* __restrict__ taps, int stride,
                                                       int dirs_per_cta, float* __restrict__ out,
                                                       int out_len, long pitch) {
  constexpr int KW = 112, W = NW * 32 * R, WPQ = NW / 4;
  constexpr int WC = R + KW;
  static_assert(WC * WPQ <= COLS, "tmem");
  extern __shared__ __align__(128) float s[];
  __shared__ unsigned tbase_s;
  float* stage_base = s + W + KW;
  int2* stp = reinterpret_cast<int2*>(stage_base + NW * 2 * 32 * R);
  const int T0 = blockIdx.x * W;
  const int d0 = blockIdx.y * dirs_per_cta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&tbase_s)), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = threadIdx.x; i < W + KW; i += NW * 32) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  for (int i = threadIdx.x; i < dirs_per_cta * stride; i += NW * 32) {
    int2 tv = taps[(long)d0 * stride + i];
    stp[i] = make_int2(KW - tv.x, tv.y);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tbase = tbase_s + ((unsigned)(32 * (warp & 3)) << 16) + (warp >> 2) * WC;
  const int tl = warp * 32 * R + lane * R;
#pragma unroll
  for (int c = 0; c < WC; c += 16) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      float4 q = *reinterpret_cast<const float4*>(&s[tl + c + i]);
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
    TLd<16>::st(v, tbase + c);
  }
  tmem_wait_st();
  float* stage = stage_base + warp * 2 * 32 * R;
  const bool full = (T0 + warp * 32 * R + 32 * R <= out_len);
  int slot = 0;
  for (int dd = 0; dd < dirs_per_cta; ++dd) {
    const int2* tp = stp + dd * stride;
    float acc[R], A[R], B[R];
    int2 cur = tp[0];
    TLd<R>::ld(A, tbase + cur.x);
#pragma unroll
    for (int k = 0; k < NNZ; ++k) {
      int2 nxt = tp[k + 1];
      tmem_wait_ld();
      float (&X)[R] = (k & 1) ? B : A;
      float (&Y)[R] = (k & 1) ? A : B;
      if (k + 1 < NNZ) TLd<R>::ld(Y, tbase + nxt.x);
      const float v = __int_as_float(cur.y);
      if (k == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = v * X[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fmaf(v, X[r], acc[r]);
      }
      cur = nxt;
    }
    float* st = stage + slot * 32 * R;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; r += 4)
      *reinterpret_cast<float4*>(st + lane * R + r) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
    __syncwarp();
    float* o = out + (d0 + dd) * pitch + T0 + warp * 32 * R;
    if (full) {
      if (lane == 0) bulk_store2(o, st, 32 * R * 4);
    } else {
      for (int i = lane; i < 32 * R; i += 32) if (T0 + warp * 32 * R + i < out_len) o[i] = st[i];
    }
    slot ^= 1;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase_s), "n"(COLS) : "memory");
}

// D) static taps (JIT-style): all offsets/values compile-time, G=4 directions per group
__device__ __forceinline__ void bulk_store(float* gdst, const float* ssrc, int bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int R>
__device__ __forceinline__ void emit(const float (&acc)[R], float* o, int SM, float* stage, int lane, int& slot, bool ok) {
  if (SM == 0) {
    if (ok) {
#pragma unroll
      for (int r = 0; r < R; r += 4)
        __stcs(reinterpret_cast<float4*>(o + r), make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]));
    }
  } else if (SM == 1) {
    float* st = stage + slot * 32 * R;
    if (lane == 0) bulk_wait_read<2>();
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; r += 4)
      *reinterpret_cast<float4*>(st + lane * R + r) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
    __syncwarp();
    if (lane == 0 && ok) bulk_store(o, st, 32 * R * 4);
    slot = (slot + 1) % 3;
  } else {
    float s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += acc[r];
    if (s == 12345.f) o[0] = s;
  }
}
template <int SM>
__global__ __launch_bounds__(128, 2) void k_static(const float* __restrict__ yf, int nyf, int dirs_per_cta,
                                                    float* __restrict__ out, int out_len, long pitch) {
  constexpr int R = 20, KW = 100, W = 128 * R;
  __shared__ __align__(128) float s[W + KW];
  __shared__ __align__(128) float stage_all[4][3][32 * R];
  const int T0 = blockIdx.x * W;
  for (int i = threadIdx.x; i < W + KW; i += 128) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tl = warp * 32 * R + lane * R;
  float win[R + KW];
#pragma unroll
  for (int i = 0; i < (R + KW) / 4; ++i) {
    float4 q = *reinterpret_cast<const float4*>(&s[tl + 4 * i]);
    win[4 * i] = q.x; win[4 * i + 1] = q.y; win[4 * i + 2] = q.z; win[4 * i + 3] = q.w;
  }
  const bool ok = (T0 + warp * 32 * R + 32 * R <= out_len);
  float* stage = &stage_all[warp][0][0];
  int slot = 0;
  const int d0 = blockIdx.y * dirs_per_cta;
  for (int dd = 0; dd < dirs_per_cta; dd += 4) {
    float* o = out + (long)(d0 + dd) * pitch + T0 + (SM == 1 ? warp * 32 * R : tl);
    float acc[R];
    asm volatile(STATIC_ASM0 : STATIC_OUTS : STATIC_INS);
    emit<R>(acc, o, SM, stage, lane, slot, ok);
    asm volatile(STATIC_ASM1 : STATIC_OUTS : STATIC_INS);
    emit<R>(acc, o + pitch, SM, stage, lane, slot, ok);
    asm volatile(STATIC_ASM2 : STATIC_OUTS : STATIC_INS);
    emit<R>(acc, o + 2 * pitch, SM, stage, lane, slot, ok);
    asm volatile(STATIC_ASM3 : STATIC_OUTS : STATIC_INS);
    emit<R>(acc, o + 3 * pitch, SM, stage, lane, slot, ok);
  }
  if (SM == 1 && lane == 0) bulk_wait_read<0>();
}
// B) smem gather: thread per output, LDS per tap
__global__ __launch_bounds__(256) void k_gather(const float* __restrict__ yf, int nyf, const int2* __restrict__ taps,
                                                int nnz, int dirs_per_cta, float* __restrict__ out, int out_len,
                                                long pitch, int KW) {
  constexpr int W = 2048;
  __shared__ float s[W + 160];
  const int T0 = blockIdx.x * W;
  for (int i = threadIdx.x; i < W + KW; i += 256) {
    int t = T0 - KW + i;
    s[i] = (t >= 0 && t < nyf) ? yf[t] : 0.f;
  }
  __syncthreads();
  const int d0 = blockIdx.y * dirs_per_cta;
  for (int d = d0; d < d0 + dirs_per_cta; ++d) {
    const int2* tp = taps + (long)d * nnz;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < nnz; ++k) {
      int2 tv = tp[k];
      float v = __int_as_float(tv.y);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fmaf(v, s[KW + threadIdx.x + 256 * j - tv.x], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int t = T0 + threadIdx.x + 256 * j;
      if (t < out_len) __stcs(out + d * pitch + t, acc[j]);
    }
  }
}

// C) FFMA throughput probe: v shared (reuse), acc/win distinct
__global__ void k_ffma(float* out, int iters, float v0) {
  float a[16], w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { a[i] = 0.f; w[i] = out[i * 64 + threadIdx.x]; }
  float v = v0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], v, w[i]);
    v += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


__global__ void k_ffma2(float* out, int iters, float v0) {
  unsigned long long a[8], w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo = threadIdx.x * 0.001f + i, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(w[i]) : "f"(lo), "f"(hi));
    a[i] = 0ull;
  }
  float v = v0;
  for (int it = 0; it < iters; ++it) {
    unsigned long long vv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(vv), "l"(w[i]));
    v += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i])); s += lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  const int ny = 441000, Lf = 101, D = 2500, nnz = 16; const int K = getenv("K52") ? 50 : 100;
  const int nyf = ny + Lf - 1, out_len = nyf + K - 1;
  const long pitch = (out_len + 31) / 32 * 32;
  std::vector<float> hyf(nyf);
  srand(1);
  for (auto& x : hyf) x = (rand() / (float)RAND_MAX) * 2 - 1;
  std::vector<int2> htaps((size_t)D * nnz);
  for (int d = 0; d < D; ++d) {
    // distinct sorted offsets
    std::vector<int> pick(K);
    for (int i = 0; i < K; ++i) pick[i] = i;
    for (int i = 0; i < nnz; ++i) { int j = i + rand() % (K - i); std::swap(pick[i], pick[j]); }
    std::vector<int> o(pick.begin(), pick.begin() + nnz);
    std::sort(o.begin(), o.end());
    for (int i = 0; i < nnz; ++i) {
      float v = fabsf((rand() / (float)RAND_MAX)) + 0.01f;
      htaps[(size_t)d * nnz + i] = make_int2(o[i], f2i(v));
    }
  }
  float *dyf, *dout;
  int2* dtaps;
  CK(cudaMalloc(&dyf, nyf * 4));
  CK(cudaMalloc(&dout, (size_t)D * pitch * 4));
  CK(cudaMalloc(&dtaps, htaps.size() * 8));
  CK(cudaMemcpy(dyf, hyf.data(), nyf * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtaps, htaps.data(), htaps.size() * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char* name) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9, sum = 0;
    for (int i = 0; i < 10; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      best = fminf(best, ms); sum += ms;
    }
    double samples = (double)D * out_len;
    printf("%-28s best %.3f ms avg %.3f ms  %.3e samples/s  %.1f GB/s write\n", name, best, sum / 10,
           samples / (best * 1e-3), samples * 4 / (best * 1e-3) / 1e9);
  };
  auto check = [&](const char* name) {
    std::vector<float> h((size_t)D * pitch);
    CK(cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int d = 0; d < D; d += 97) {
      for (int t = 0; t < out_len; t += 7) {
        double ref = 0;
        for (int k = 0; k < nnz; ++k) {
          int2 tv = htaps[(size_t)d * nnz + k];
          int s = t - tv.x;
          if (s >= 0 && s < nyf) ref += (double)i2f(tv.y) * hyf[s];
        }
        maxerr = fmax(maxerr, fabs(ref - h[(size_t)d * pitch + t]));
      }
    }
    printf("  %s maxabs err %.3e\n", name, maxerr);
  };
  std::vector<int2> htaps2((size_t)D * (nnz + 1));
  for (int d = 0; d < D; ++d) {
    for (int i = 0; i < nnz; ++i) htaps2[(size_t)d * (nnz + 1) + i] = htaps[(size_t)d * nnz + i];
    htaps2[(size_t)d * (nnz + 1) + nnz] = make_int2(getenv("K52") ? 52 : 100, 0);
  }
  int2* dtaps2; CK(cudaMalloc(&dtaps2, htaps2.size() * 8));
  CK(cudaMemcpy(dtaps2, htaps2.data(), htaps2.size() * 8, cudaMemcpyHostToDevice));
  const char* only = getenv("ONLY");
  for (int dpc : {125}) {
#define RUNV(R_, MINB_, V_) { constexpr int R = R_; dim3 grid((out_len + 128 * R - 1) / (128 * R), D / dpc); \
      size_t sm = (128 * R + V_ + 28 + 4 * 3 * 32 * R) * 4 + dpc * (nnz + 1) * 8; \
      cudaFuncSetAttribute(k_jtasm2<R, MINB_, V_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
      char nm[64]; snprintf(nm, 64, "jtasm2 KW=%d R=%d minb=%d dpc=%d", V_, R, MINB_, dpc); \
      timeit([&] { k_jtasm2<R, MINB_, V_><<<grid, 128, sm>>>(dyf, nyf, dtaps2, nnz + 1, dpc, dout, out_len, pitch); }, nm); \
      check(nm); }
    if (getenv("K52")) { RUNV(20, 3, 52) RUNV(36, 2, 52) RUNV(12, 4, 52) } else { RUNV(20, 3, 100) RUNV(12, 3, 100) RUNV(28, 2, 100) }
    if (only) break;
    }
  if (getenv("TMEM")) {
    int dpc = 125;
#define RUNT(RB_, NW_, COLS_, MINB_) { constexpr int R = 16 * RB_; dim3 grid((out_len + NW_ * 32 * R - 1) / (NW_ * 32 * R), D / dpc); \
      size_t sm = (NW_ * 32 * R + 100 + 28 + NW_ * 3 * 32 * R) * 4 + dpc * (nnz + 1) * 8; \
      CK(cudaFuncSetAttribute(k_tmem<RB_, NW_, COLS_, MINB_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
      char nm[64]; snprintf(nm, 64, "tmem R=%d NW=%d cols=%d", R, NW_, COLS_); \
      timeit([&] { k_tmem<RB_, NW_, COLS_, MINB_><<<grid, NW_ * 32, sm>>>(dyf, nyf, dtaps2, nnz + 1, dpc, dout, out_len, pitch); }, nm); \
      CK(cudaGetLastError()); check(nm); }
    RUNT(1, 4, 128, 4)
    RUNT(1, 8, 256, 2)
    RUNT(2, 4, 256, 2)
    RUNT(2, 8, 512, 1)
  }
  if (getenv("TMEM2")) {
#define RUNT2(R_, NW_, COLS_, MINB_, DPC_) { constexpr int R = R_; int dpc = DPC_; dim3 grid((out_len + NW_ * 32 * R - 1) / (NW_ * 32 * R), D / dpc); \
      size_t sm = (NW_ * 32 * R + 112 + NW_ * 2 * 32 * R) * 4 + dpc * (nnz + 1) * 8; \
      CK(cudaFuncSetAttribute(k_tmem2<R_, NW_, COLS_, MINB_, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
      char nm[64]; snprintf(nm, 64, "tmem2 R=%d NW=%d cols=%d dpc=%d", R, NW_, COLS_, dpc); \
      timeit([&] { k_tmem2<R_, NW_, COLS_, MINB_, 16><<<grid, NW_ * 32, sm>>>(dyf, nyf, dtaps2, nnz + 1, dpc, dout, out_len, pitch); }, nm); \
      CK(cudaGetLastError()); check(nm); }
    RUNT2(16, 4, 128, 4, 125)
    RUNT2(16, 4, 128, 4, 50)
    RUNT2(16, 16, 512, 1, 125)
    RUNT2(32, 12, 512, 1, 125)
    RUNT2(32, 12, 512, 1, 50)
  }
  if (getenv("STATIC")) {
    for (int dpc : {20, 100}) {
      dim3 grid((out_len + 128 * 20 - 1) / (128 * 20), D / dpc);
      char nm[64];
      snprintf(nm, 64, "static stg R=20 dpc=%d", dpc);
      timeit([&] { k_static<0><<<grid, 128>>>(dyf, nyf, dpc, dout, out_len, pitch); }, nm);
      snprintf(nm, 64, "static bulk R=20 dpc=%d", dpc);
      timeit([&] { k_static<1><<<grid, 128>>>(dyf, nyf, dpc, dout, out_len, pitch); }, nm);
      snprintf(nm, 64, "static nostore R=20 dpc=%d", dpc);
      timeit([&] { k_static<2><<<grid, 128>>>(dyf, nyf, dpc, dout, out_len, pitch); }, nm);
    }
  }
  if (only) return 0;
  // memset roofline
  timeit([&] { cudaMemsetAsync(dout, 0, (size_t)D * pitch * 4); }, "memset out");
  // FFMA probe
  {
    float* dd; CK(cudaMalloc(&dd, 148 * 8 * 256 * 4));
    int iters = 20000;
    for (int i = 0; i < 2; ++i) k_ffma<<<148 * 8, 256>>>(dd, iters, 1.0f);
    cudaEventRecord(e0);
    k_ffma<<<148 * 8, 256>>>(dd, iters, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 148 * 8 * 256 * (double)iters * 16;
    printf("FFMA probe: %.3f ms  %.2f TFLOP/s\n", ms, fl / (ms * 1e-3) / 1e12);
  }
  {
    float* dd; CK(cudaMalloc(&dd, 148 * 8 * 256 * 4));
    int iters = 20000;
    for (int i = 0; i < 2; ++i) k_ffma2<<<148 * 8, 256>>>(dd, iters, 1.0f);
    cudaEventRecord(e0);
    k_ffma2<<<148 * 8, 256>>>(dd, iters, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 148 * 8 * 256 * (double)iters * 16;
    printf("FFMA2 probe: %.3f ms  %.2f TFLOP/s\n", ms, fl / (ms * 1e-3) / 1e12);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz\n", clk);
  return 0;
}
