// Tensor-core renderer: out[e][d] = (y * f_e) * g_{e,d} with stage 2 as a GEMM
// on the 5th-generation tensor cores (tcgen05.mma kind::f16, fp32 accumulate
// in TMEM).
//
// Reference semantics: toepnmf Renderer.render (pkg/src/toepnmf/engine/__init__.py:238-260)
// = conv_dense(y, f) (_kernels.pyx:11-25) then conv_sparse(yf, idx, vals, K)
// (_kernels.pyx:28-44), for every (ear, direction) row.
//
// Stage 2 for a tile of 128 outputs t and a chunk of 64 directions d is
//     D[t][d] = sum_o A[t][o] * G[d][o],   A[t][o] = yf[T0 + t - o]   (Toeplitz/Hankel)
// with o < KPAD = round_up(K, 16): M = 128, N = 64, K = KPAD.  The zero taps of
// the sparse g cost tensor-core work, but the tensor cores have ~2x headroom
// over the HBM write stream at every sparsity (the kernel is write-bound).
//
// fp32 accuracy from fp16 operands: x = hi + lo with hi = fp16(x),
// lo = fp16(x - hi) (exact residual), products hi*hi + hi*lo + lo*hi in fp32
// (the dropped lo*lo term is ~2^-22 relative).  Operands are scaled by powers
// of two into [2^13, 2^14) before the split -- per tile for yf, per direction
// for g -- and unscaled exactly in the epilogue, so the split never meets
// fp16 under/overflow.  Measured rel. L2 ~6e-7 (tools/microbench/mma_probe.cu).
//
// Persistent, warp-specialised CTA (one per SM, 16 warps):
//   warp 0      : TMA producer -- G chunks (pre-laid-out canonical fp16 hi/lo,
//                 32 KB for KPAD 128) into a 2-deep ring (cp.async.bulk + mbarrier)
//   warp 1      : MMA issuer (one elected lane): per chunk 3 x KPAD/16
//                 tcgen05.mma per t-tile into a double-buffered TMEM accumulator
//   warps 2-7   : A builders -- stage 1 (resonance FIR) for the item's yf tile,
//                 the per-tile scale, and the Hankel A tile in the canonical
//                 K-major layout (hi and lo), once per item (TT x 128 outputs)
//   warps 8-15  : epilogue -- tcgen05.ld the accumulator (lane = output t; two
//                 warps per lane quarter, 32 columns each), unscale, stage a
//                 [32 directions][32 t] block in shared memory, TMA tensor store
//                 (3-D map {t, direction, ear} clips the padding directions)
#include <algorithm>
#include <cstdio>
#include <cuda_fp16.h>

#include "common.cuh"
#include "launch.h"

namespace toep {

#ifndef TOEP_MMA_NOMMA
#define TOEP_MMA_NOMMA 0
#endif
#ifndef TOEP_MMA_PROF
#define TOEP_MMA_PROF 0
#endif
#if TOEP_MMA_PROF
#define PW(slot, ...)                \
  do {                               \
    const long long _t0 = clock64(); \
    __VA_ARGS__;                     \
    prof[slot] += clock64() - _t0;   \
  } while (0)
#else
#define PW(slot, ...) __VA_ARGS__
#endif
constexpr int kMmaM = 128;        // outputs per t-tile
constexpr int kMmaN = 64;         // directions per chunk
constexpr int kMmaBuilderWarps = 6;
constexpr int kMmaEpiWarps = 8;  // two per TMEM lane quarter (32 columns each)
constexpr int kMmaWarps = 2 + kMmaBuilderWarps + kMmaEpiWarps;
constexpr int kMmaThreads = 32 * kMmaWarps;
constexpr int kMmaBuilders = 32 * kMmaBuilderWarps;

// byte offset of element (r, k) in an R-row, K-major, SWIZZLE_NONE canonical
// operand: 8x16-byte core matrices, rows of a core at 16 B, the two K halves
// of a 16-wide k-step at LBO = 128 B, 8-row groups at SBO = 256 B, k-steps at R*32 B
__host__ __device__ inline int mma_canon(int r, int k, int R) {
  return (k >> 4) * (R * 32) + (r >> 3) * 256 + ((k >> 3) & 1) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t mma_sdesc(unsigned saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

__device__ __forceinline__ void mma_f16(unsigned d_tmem, uint64_t da, uint64_t db, uint32_t idesc, int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void builders_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMmaBuilders) : "memory"); }

__device__ __forceinline__ unsigned pack_half2(__half a, __half b) {
  return (unsigned)__half_as_ushort(a) | ((unsigned)__half_as_ushort(b) << 16);
}

struct MmaSmem {
  int a_off, b_off, st_off, y_off, yf_off, f_off, red_off, sc_off, bars_off, total;
};

__host__ __device__ inline MmaSmem mma_smem(int kpad, int tt, int lf_pad) {
  MmaSmem L{};
  const int a_bytes = tt * 2 * kMmaM * kpad * 2;
  const int b_bytes = 2 * 2 * kMmaN * kpad * 2;
  L.a_off = 0;
  L.b_off = a_bytes;
  int off = a_bytes + b_bytes;  // floats from here (all offsets in bytes)
  L.st_off = off;               // epilogue staging: [epilogue warps][32 directions][32 t]
  off += kMmaEpiWarps * 32 * 32 * 4;
  L.y_off = off;
  off += ((kMmaM * tt + kpad + lf_pad + 31) & ~31) * 4;
  L.yf_off = off;
  off += ((kMmaM * tt + kpad + 31) & ~31) * 4;
  L.f_off = off;
  off += ((lf_pad + 31) & ~31) * 4;
  L.red_off = off;
  off += 32 * 4;
  L.sc_off = off;
  off += 8 * 4;
  L.bars_off = off;
  off += 16 * 8;
  L.total = off + 1024;  // alignment slack
  return L;
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const float* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tm),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

__global__ void __launch_bounds__(kMmaThreads, 1)
    k_render_mma(RenderMmaArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  const int TT = a.tt, KP = a.kpad, KS = KP / 16;
  const MmaSmem L = mma_smem(KP, TT, a.lf_pad);
  const int a_part_bytes = kMmaM * KP * 2;
  const int b_part_bytes = kMmaN * KP * 2;
  const int b_chunk_bytes = 2 * b_part_bytes;
  unsigned char* sA = sm + L.a_off;  // [TT][hi, lo][canonical 128 x KP]
  unsigned char* sB = sm + L.b_off;  // [2 stages][hi, lo][canonical 64 x KP]
  float* s_y = reinterpret_cast<float*>(sm + L.y_off);
  float* s_yf = reinterpret_cast<float*>(sm + L.yf_off);
  float* s_f = reinterpret_cast<float*>(sm + L.f_off);
  float* s_red = reinterpret_cast<float*>(sm + L.red_off);
  float* s_sc = reinterpret_cast<float*>(sm + L.sc_off);  // per item (ring of 2): 2^-s
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars_off);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* b_full = bars + 2;       // [2]
  uint64_t* b_empty = bars + 4;      // [2]
  uint64_t* acc_full = bars + 6;     // [2]
  uint64_t* acc_empty = bars + 8;    // [2]
  uint64_t* sc_full = bars + 10;     // [2]
  uint64_t* sc_empty = bars + 12;    // [2]
  __shared__ unsigned s_tbase;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if TOEP_MMA_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif
  if (warp == 0) tmem_alloc<256>(&s_tbase);
  if (tid == 32) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kMmaEpiWarps);
      mbar_init(&sc_full[i], 1);
      mbar_init(&sc_empty[i], kMmaEpiWarps);
    }
    mbar_fence_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tbase = s_tbase;

  const long long u0 = a.n_units * blockIdx.x / gridDim.x;
  const long long u1 = a.n_units * (blockIdx.x + 1) / gridDim.x;
  const int nch = a.nchunks;

  if (warp == 0) {
    // ===== G chunk producer =====
    if (elect_one()) {
      int bs = 0;
      unsigned bph = 0;
      const unsigned char* g = reinterpret_cast<const unsigned char*>(a.g);
      for (long long u = u0; u < u1; ++u) {
        const int c = (int)(u % nch);
        const int e = (int)(u / nch / a.n_titems);
        PW(0, mbar_wait_sleep(&b_empty[bs], bph ^ 1u));
        mbar_arrive_expect_tx(&b_full[bs], (unsigned)b_chunk_bytes);
        bulk_load(sB + bs * b_chunk_bytes, g + ((long long)e * nch + c) * b_chunk_bytes, (unsigned)b_chunk_bytes,
                  &b_full[bs]);
        if (++bs == 2) {
          bs = 0;
          bph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(kMmaN >> 3) << 17) | ((uint32_t)(kMmaM >> 4) << 24);
      int bs = 0, as = 0;
      unsigned bph = 0, aph = 0, a_ph = 0;
      long long cur = -1;
      const unsigned sa = smem_u32(sA), sb = smem_u32(sB);
      for (long long u = u0; u < u1; ++u) {
        const long long item = u / nch;
        if (item != cur) {
          if (cur >= 0) mma_commit(a_empty);  // A of the previous item is free once its MMAs retire
          PW(1, mbar_wait_sleep(a_full, a_ph));
          a_ph ^= 1u;
          cur = item;
        }
        PW(2, mbar_wait_sleep(&b_full[bs], bph));
        PW(3, mbar_wait_sleep(&acc_empty[as], aph ^ 1u));
        tmem_fence_after();
        for (int tt = 0; tt < TT; ++tt) {
          const unsigned d = tbase + (unsigned)(as * TT * kMmaN + tt * kMmaN);
          int acc = 0;
#pragma unroll 1
          for (int p = 0; p < 3; ++p) {  // hi*hi, hi*lo, lo*hi
            const unsigned pa = sa + (unsigned)((tt * 2 + (p == 2 ? 1 : 0)) * a_part_bytes);
            const unsigned pb = sb + (unsigned)(bs * b_chunk_bytes + (p == 1 ? 1 : 0) * b_part_bytes);
            for (int ks = 0; ks < KS; ++ks) {
#if !TOEP_MMA_NOMMA
              mma_f16(d, mma_sdesc(pa + ks * kMmaM * 32), mma_sdesc(pb + ks * kMmaN * 32), idesc, acc);
#endif
              acc = 1;
            }
          }
        }
        mma_commit(&b_empty[bs]);
        mma_commit(&acc_full[as]);
        if (++bs == 2) {
          bs = 0;
          bph ^= 1u;
        }
        if (++as == 2) {
          as = 0;
          aph ^= 1u;
        }
      }
    }
  } else if (warp < 2 + kMmaBuilderWarps) {
    // ===== A builders: stage 1 + Hankel operand =====
    const int bt = tid - 64;
    const int YF = kMmaM * TT + KP - 1;  // yf samples of an item
    const int YL = YF + a.lf_pad - 1;    // y samples feeding them
    unsigned a_ph = 0;
    long long cur = -1;
    int cur_e = -1, nitem = 0;
    float chk = 0.f;
    for (long long u = u0; u < u1; ++u) {
      const long long item = u / nch;
      if (item == cur) continue;
      cur = item;
      const int ti = (int)(item % a.n_titems), e = (int)(item / a.n_titems);
      const long long T0 = (long long)ti * kMmaM * TT;
      const long long y0 = T0 - (KP - 1) - (a.lf_pad - 1);
      PW(4, mbar_wait_sleep(a_empty, a_ph ^ 1u));  // MMAs of the previous item retired (first pass: free)
      a_ph ^= 1u;
      if (e != cur_e)
        for (int i = bt; i < a.lf_pad; i += kMmaBuilders) s_f[i] = a.f[(long long)e * a.lf_pad + i];
      cur_e = e;
      for (int i = bt; i < YL; i += kMmaBuilders) {
        const long long t = y0 + i;
        const float v = (t >= 0 && t < a.nx) ? __ldg(a.x + t) : 0.f;
        chk = fmaf(v, 0.f, chk);
        s_y[i] = v;
      }
      builders_sync();
      float mx = 0.f;
      for (int i = bt; i < YF; i += kMmaBuilders) {
        float acc = 0.f;
        const float* yy = s_y + i + a.lf_pad - 1;
        for (int j = 0; j < a.lf_pad; ++j) acc = fmaf(s_f[j], yy[-j], acc);
        s_yf[i] = acc;
        mx = fmaxf(mx, fabsf(acc));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) s_red[warp - 2] = mx;
      builders_sync();
      mx = 0.f;
      for (int w = 0; w < kMmaBuilderWarps; ++w) mx = fmaxf(mx, s_red[w]);
      const int sexp = mx > 0.f ? 13 - ilogbf(mx) : 0;  // max |yf| * 2^sexp in [2^13, 2^14)
      const float scale = ldexpf(1.f, sexp);
      if (bt == 0) {
        mbar_wait_sleep(&sc_empty[nitem & 1], (unsigned)(((nitem >> 1) & 1) ^ 1));
        s_sc[nitem & 1] = ldexpf(1.f, -sexp);
        mbar_arrive(&sc_full[nitem & 1]);
      }
      // Hankel A: entry (tt, t, kc) = yf[T0 + 128 tt + t - o], o = 8 kc .. 8 kc + 7
      const int KC = KP / 8;
#pragma unroll 1
      for (int idx = bt; idx < TT * kMmaM * KC; idx += kMmaBuilders) {
        const int t = idx & (kMmaM - 1);
        const int rest = idx >> 7;
        const int kc = rest % KC, tt = rest / KC;
        const float* src = s_yf + (kMmaM * tt + t + KP - 1) - 8 * kc;
        unsigned hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float x0 = src[-i] * scale, x1 = src[-i - 1] * scale;
          const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
          const __half l0 = __float2half_rn(x0 - __half2float(h0)), l1 = __float2half_rn(x1 - __half2float(h1));
          hw[i / 2] = pack_half2(h0, h1);
          lw[i / 2] = pack_half2(l0, l1);
        }
        const int off = mma_canon(t, 8 * kc, kMmaM);
        *reinterpret_cast<uint4*>(sA + (tt * 2 + 0) * a_part_bytes + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(sA + (tt * 2 + 1) * a_part_bytes + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
      builders_sync();
      if (bt == 0) mbar_arrive(a_full);
      ++nitem;
    }
    if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
  } else {
    // ===== epilogue: TMEM -> registers -> HBM =====
    const int q = warp & 3;                                   // TMEM lane quarter of this warp
    const int half = (warp - 2 - kMmaBuilderWarps) >> 2;      // which 32 of the chunk's 64 columns
    float* stg = reinterpret_cast<float*>(sm + L.st_off) + (warp - 2 - kMmaBuilderWarps) * 32 * 32;
    const unsigned tq = tbase + ((unsigned)(32 * q) << 16);
    int as = 0;
    unsigned aph = 0;
    long long cur = -1;
    int nitem = -1;
    float unscale = 1.f;
    for (long long u = u0; u < u1; ++u) {
      const long long item = u / nch;
      const int c = (int)(u % nch);
      const int ti = (int)(item % a.n_titems), e = (int)(item / a.n_titems);
      if (item != cur) {
        if (nitem >= 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sc_empty[nitem & 1]);
        }
        ++nitem;
        mbar_wait_sleep(&sc_full[nitem & 1], (unsigned)((nitem >> 1) & 1));
        unscale = s_sc[nitem & 1];
        cur = item;
      }
      PW(5, mbar_wait_sleep(&acc_full[as], aph));
      tmem_fence_after();
      const long long T0 = (long long)ti * kMmaM * TT;
      const int d0 = c * kMmaN + 32 * half;  // this warp's 32 directions of the chunk
      // per-direction unscale for the warp's 32 columns: lane j holds column j's factor
      const float gsl = (d0 + lane < a.dirs ? __ldg(a.gscale + (long long)e * a.dirs_pad + d0 + lane) : 0.f) * unscale;
#pragma unroll 1
      for (int tt = 0; tt < TT; ++tt) {
        const long long t0 = T0 + kMmaM * tt + 32 * q;
        if (t0 >= a.out_len) continue;
        if (lane == 0) bulk_wait_read<0>();  // the previous store has read the staging block
        __syncwarp();
#pragma unroll
        for (int cb = 0; cb < 32; cb += 16) {
          float v[16];
          tmem_ld16(v, tq + (unsigned)(as * TT * kMmaN + tt * kMmaN + 32 * half + cb));
          tmem_wait_ld();
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) stg[(cb + jj) * 32 + lane] = v[jj] * __shfl_sync(0xffffffffu, gsl, cb + jj);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (elect_one()) {
          tma_store_3d(&tm, stg, (int)t0, d0, e);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      tmem_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[as]);
      if (++as == 2) {
        as = 0;
        aph ^= 1u;
      }
    }
  }
  if (warp >= 2 + kMmaBuilderWarps && lane == 0) bulk_wait_all();
#if TOEP_MMA_PROF
  if (blockIdx.x == 7 && lane == 0 && (warp <= 2 || warp == 8))
    printf("prof cta7 warp %d total %lld: b_empty %lld a_full %lld b_full %lld acc_empty %lld a_empty %lld acc_full %lld\n",
           warp, clock64() - t_start, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5]);
#endif
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

// G[e][c] chunk = [hi, lo][canonical 64 x kpad] fp16 of the dense rows of
// directions 64c .. 64c+63, each row scaled by 2^q (max |g| * 2^q in
// [2^13, 2^14)); gscale[e][d] = 2^-q.  One warp per (ear, direction) row.
__global__ void k_build_gmma(const int2* __restrict__ raw, const int* __restrict__ nnz, int dirs, int ears,
                             int stride, int kpad, int nchunks, int dirs_pad, __half* __restrict__ g,
                             float* __restrict__ gscale) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= ears * dirs) return;
  const int e = row / dirs, d = row - e * dirs;
  const int n = nnz[row];
  const int2* taps = raw + (long long)row * stride;
  float mx = 0.f;
  for (int k = lane; k < n; k += 32) mx = fmaxf(mx, fabsf(__int_as_float(taps[k].y)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int qexp = mx > 0.f ? 13 - ilogbf(mx) : 0;
  if (lane == 0) gscale[(long long)e * dirs_pad + d] = ldexpf(1.f, -qexp);
  const int c = d / kMmaN, r = d - c * kMmaN;
  unsigned char* base = reinterpret_cast<unsigned char*>(g) + ((long long)e * nchunks + c) * 2 * kMmaN * kpad * 2;
  for (int k = 0; k < n; ++k) {  // taps are unique offsets; everything else stays zero (memset)
    if (lane != 0) break;
    const int o = taps[k].x;
    const float x = ldexpf(__int_as_float(taps[k].y), qexp);
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *reinterpret_cast<__half*>(base + mma_canon(r, o, kMmaN)) = h;
    *reinterpret_cast<__half*>(base + kMmaN * kpad * 2 + mma_canon(r, o, kMmaN)) = l;
  }
}

int render_mma_kpad(int K) { return (K + 15) / 16 * 16; }
int render_mma_tt(int kpad) { return kpad <= 128 ? 2 : 1; }

bool render_mma_supported(int K, int lf_pad) {
  const int kp = render_mma_kpad(K);
  if (kp > 192 || lf_pad > 512) return false;
  return mma_smem(kp, render_mma_tt(kp), lf_pad).total <= 227 * 1024;
}

size_t render_mma_gbytes(int ears, int dirs, int K) {
  const int kp = render_mma_kpad(K);
  const int nch = (dirs + kMmaN - 1) / kMmaN;
  return (size_t)ears * nch * 2 * kMmaN * kp * 2;
}

cudaError_t build_render_mma_tables(const int2* raw, const int* nnz, int dirs, int ears, int stride, int K,
                                    void* g, float* gscale, cudaStream_t st) {
  const int kp = render_mma_kpad(K);
  const int nch = (dirs + kMmaN - 1) / kMmaN;
  cudaError_t e = cudaMemsetAsync(g, 0, render_mma_gbytes(ears, dirs, K), st);
  if (e != cudaSuccess) return e;
  const int rows = ears * dirs;
  k_build_gmma<<<(rows + 7) / 8, 256, 0, st>>>(raw, nnz, dirs, ears, stride, kp, nch, nch * kMmaN,
                                               reinterpret_cast<__half*>(g), gscale);
  return cudaGetLastError();
}

cudaError_t launch_render_mma(const RenderMmaArgs& a, const CUtensorMap& map, int sm_count, cudaStream_t st) {
  const MmaSmem L = mma_smem(a.kpad, a.tt, a.lf_pad);
  cudaError_t err = cudaFuncSetAttribute(k_render_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  if (err != cudaSuccess) return err;
  long long grid = std::min<long long>(sm_count, a.n_units);
  if (grid < 1) return cudaSuccess;
  k_render_mma<<<(unsigned)grid, kMmaThreads, L.total, st>>>(a, map);
  return cudaGetLastError();
}

}  // namespace toep
