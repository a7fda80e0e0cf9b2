// Tensor-core renderer: out[e][d] = (y * f_e) * g_{e,d} with stage 2 as a GEMM
// on the 5th-generation tensor cores (tcgen05.mma kind::f16, fp32 accumulate
// in TMEM).
//
// Reference semantics: toepnmf Renderer.render (pkg/src/toepnmf/engine/__init__.py:238-260)
// = conv_dense(y, f) (_kernels.pyx:11-25) then conv_sparse(yf, idx, vals, K)
// (_kernels.pyx:28-44), for every (ear, direction) row.
//
// Stage 2 for a tile of 128 outputs t and a chunk of 128 directions d is
//     D[t][d] = sum_o A[t][o] * G[d][o],   A[t][o] = yf[T0 + t - o]   (Hankel)
// with o < KPAD = round_up(K, 16): M = N = 128, K = KPAD (an M=128 MMA costs
// the same ~64 cycles at N = 64 as at N = 128, so N = 128 runs at full rate).
// The zero taps of the sparse g cost tensor-core work, but the tensor cores
// have ~2x headroom over the HBM write stream at every sparsity: the kernel
// is write-bound.
//
// fp32 accuracy from fp16 operands: x = hi + lo with hi = fp16(x),
// lo = fp16(x - hi) (exact residual), products hi*hi + hi*lo + lo*hi in fp32
// (the dropped lo*lo term is ~2^-22 relative).  Operands are scaled by powers
// of two into [2^13, 2^14) before the split -- per 128-output tile for yf, per
// 128-direction chunk for g -- and unscaled exactly in the epilogue, so the
// split never meets fp16 under/overflow.  Measured rel. L2 2e-7..1e-6
// (tests/test_gpu_paths.py; tools/microbench/mma_probe.cu).
//
// The Hankel operand A lives in TMEM (lane t = output t, column j = the fp16
// pair {A[t][2j], A[t][2j+1]}), so each MMA reads only G from shared memory
// (with A in shared memory the MMAs were shared-memory-bandwidth bound); two
// A buffers when KPAD <= 128, so the next tile's rows are written while this
// tile's MMAs run (at KPAD 160 the hi / lo halves rotate through three TMEM
// slots instead).  G chunks are shared by a cluster of CL CTAs that render
// consecutive tiles in lockstep: each CTA loads 1/CL of every chunk with a
// multicast bulk copy, and each CTA's MMA completion frees the stage in all
// of them (tcgen05.commit .multicast::cluster).  A render is one launch of
// 6-CTA clusters (22 fit a B200's GPCs: 132 SMs) plus a concurrent launch of
// 2-CTA clusters on the 16 SMs left, each over its own share of every ear's
// tiles (launch_render_mma).
//
// Persistent, warp-specialised CTA (one per SM, 18 warps):
//   warp 0      : TMA producer -- its slice of each G chunk (canonical fp16
//                 hi/lo, 57 KB per chunk at KPAD 112) into a 2-stage ring
//   warp 1      : MMA issuer (one elected lane): per unit 3 x KPAD/16
//                 tcgen05.mma (A from TMEM, G from shared memory) into a
//                 double-buffered TMEM accumulator
//   warps 2-9   : A builders -- stage 1 (resonance FIR) for the tile's yf,
//                 the tile scale, then every thread writes its TMEM lane's
//                 Hankel row (hi and lo) with tcgen05.st; once per tile
//   warps 10-17 : epilogue -- tcgen05.ld the accumulator (lane = output t; two
//                 warps per lane quarter, 64 columns each), unscale, stage
//                 [32 directions][32 t] blocks in shared memory, TMA tensor
//                 stores (3-D map {t, direction, ear} clips padding directions)
#include <algorithm>
#include <climits>
#include <mutex>
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
// 2^e for e in [-126, 127] (exact; callers split larger exponents in two);
// clamped at the ends, where the product they scale under/overflows anyway
__device__ __forceinline__ float exp2i(int e) { return __int_as_float((127 + max(-126, min(127, e))) << 23); }
constexpr int kMmaM = 128;        // outputs per t-tile
constexpr int kMmaN = 128;        // directions per chunk (M = 128, N = 128: full tensor rate, N = 64 runs at half)
constexpr int kMmaBuilderWarps = 8;  // two per TMEM lane quarter
constexpr int kMmaEpiWarps = 8;      // two per TMEM lane quarter (64 columns each)
constexpr int kMmaWarps = 2 + kMmaBuilderWarps + kMmaEpiWarps;
constexpr int kMmaThreads = 32 * kMmaWarps;
constexpr int kMmaBuilders = 32 * kMmaBuilderWarps;
#ifndef TOEP_MMA_BSTAGES
#define TOEP_MMA_BSTAGES 2
#endif
constexpr int kMmaBStages = TOEP_MMA_BSTAGES;

#ifndef TOEP_MMA_CLUSTER
#define TOEP_MMA_CLUSTER 6
#endif
constexpr int kMmaCluster = TOEP_MMA_CLUSTER;  // CTAs sharing each G chunk load (TMA multicast); 6 measured best of 1-8
constexpr int kMmaAccCols = 2 * kMmaN;  // accumulators: 2 buffers x 128 columns; A buffers follow

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

// D[tmem] (+)= A[tmem] * B[smem]^T, fp16 inputs, fp32 accumulate
__device__ __forceinline__ void mma_f16_ts(unsigned d_tmem, unsigned a_tmem, uint64_t db, uint32_t idesc,
                                           int accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned num_clusters_x() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 1-D bulk copy global -> the same shared-memory offset of every CTA in `mask`,
// completion counted on each destination CTA's mbarrier at `bar`'s offset
__device__ __forceinline__ void bulk_load_multicast(void* sdst, const void* gsrc, unsigned bytes, uint64_t* bar,
                                                    unsigned short mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// MMA completion -> arrive on the barrier at `bar`'s offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_multicast(uint64_t* bar, unsigned short mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}

__device__ __forceinline__ void builders_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kMmaBuilders) : "memory"); }

__device__ __forceinline__ unsigned pack_half2(__half a, __half b) {
  return (unsigned)__half_as_ushort(a) | ((unsigned)__half_as_ushort(b) << 16);
}

__device__ __forceinline__ void tmem_st8(unsigned ta, const unsigned (&w)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, const float* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tm),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

struct MmaSmem {
  int b_off, st_off, y_off, yf_off, f_off, red_off, sc_off, fac_off, bars_off, total, nstg;
};

__host__ __device__ inline MmaSmem mma_smem_n(int kpad, int lf_pad, int nstg) {
  MmaSmem L{};
  L.b_off = 0;  // [kMmaBStages][hi, lo][canonical 128 x kpad] fp16
  int off = kMmaBStages * 2 * kMmaN * kpad * 2;
  L.st_off = off;  // epilogue staging: [epilogue warps][nstg buffers][32 directions][32 t] fp32
  off += kMmaEpiWarps * nstg * 32 * 32 * 4;
  L.y_off = off;
  off += ((kMmaM + kpad + lf_pad + 31) & ~31) * 4;
  L.yf_off = off;
  off += ((kMmaM + kpad + 31) & ~31) * 4;
  L.f_off = off;
  off += ((lf_pad + 31) & ~31) * 4;
  L.red_off = off;
  off += 32 * 4;
  L.sc_off = off;
  off += 8 * 4;
  L.fac_off = off;  // wide G chunks: per-column unscale factors [epilogue warps][2][64]
  off += kMmaEpiWarps * 2 * 64 * 4;
  L.bars_off = off;
  off += (12 + 2 * kMmaBStages + 5) * 8;
  L.total = off + 1024;  // alignment slack
  L.nstg = nstg;
  return L;
}

// double-buffered epilogue staging when it fits next to the G ring, else single
__host__ __device__ inline MmaSmem mma_smem(int kpad, int lf_pad) {
  const MmaSmem L2 = mma_smem_n(kpad, lf_pad, 2);
  return L2.total <= 227 * 1024 ? L2 : mma_smem_n(kpad, lf_pad, 1);
}

// A buffers in TMEM after the two accumulators: two when they fit (the next
// item's Hankel rows are written while this item's MMAs run), else one
__host__ __device__ inline int mma_a_buffers(int kpad) { return kMmaAccCols + 2 * kpad <= 512 ? 2 : 1; }

template <int CL>
__global__ void __launch_bounds__(kMmaThreads, 1)
    k_render_mma(RenderMmaArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  const int KP = a.kpad, KS = KP / 16, NA = mma_a_buffers(KP);
  const bool ring = NA == 1 && kMmaAccCols + 3 * (KP / 2) <= 512;
  const MmaSmem L = mma_smem(KP, a.lf_pad);
  const int b_part_bytes = kMmaN * KP * 2;
  const int b_chunk_bytes = 2 * b_part_bytes;
  unsigned char* sB = sm + L.b_off;
  float* s_y = reinterpret_cast<float*>(sm + L.y_off);
  float* s_yf = reinterpret_cast<float*>(sm + L.yf_off);
  float* s_f = reinterpret_cast<float*>(sm + L.f_off);
  float* s_red = reinterpret_cast<float*>(sm + L.red_off);
  float* s_sc = reinterpret_cast<float*>(sm + L.sc_off);  // per item (ring of 2): 2^-s
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars_off);
  uint64_t* a_full = bars + 0;     // [2]
  uint64_t* a_empty = bars + 2;    // [2]
  uint64_t* acc_full = bars + 4;   // [2]
  uint64_t* acc_empty = bars + 6;  // [2]
  uint64_t* sc_full = bars + 8;    // [2]
  uint64_t* sc_empty = bars + 10;  // [2]
  uint64_t* b_full = bars + 12;    // [kMmaBStages]
  uint64_t* b_empty = b_full + kMmaBStages;
  // ring mode (one A buffer does not leave room for two): hi and lo halves of
  // successive items rotate through three KP/2-column slots; item i's hi goes
  // to slot (2i) % 3 and its lo to (2i+1) % 3, so the next item's hi is written
  // while this item runs and its lo as soon as this item's hi MMAs retire.
  // a_full doubles as hi_full.
  uint64_t* lo_full = b_empty + kMmaBStages;  // [2]
  uint64_t* slot_free = lo_full + 2;          // [3]
  __shared__ unsigned s_tbase;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if TOEP_MMA_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
#endif
  if (warp == 0) tmem_alloc<512>(&s_tbase);
  if (tid == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 1);
      mbar_init(&a_empty[i], 1);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kMmaEpiWarps);
      mbar_init(&sc_full[i], 1);
      mbar_init(&sc_empty[i], kMmaEpiWarps);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&lo_full[i], 1);
    for (int i = 0; i < 3; ++i) mbar_init(&slot_free[i], 1);
    for (int i = 0; i < kMmaBStages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], CL);  // every CTA of the cluster frees the stage
    }
    mbar_fence_init();
  }
  tmem_fence_before();
  cluster_sync_all();  // barrier inits visible cluster-wide before any multicast lands
  tmem_fence_after();
  const unsigned tbase = s_tbase;

  // Work: groups of kMmaCluster consecutive 128-output tiles of one ear; the
  // cluster walks a contiguous range of groups, CTA `crank` renders tile
  // 4*group + crank of each, all CTAs stepping through the same G chunks in
  // lockstep (unit = (group, chunk)).  Tiles past the end render zeros and
  // store nothing.
  const int nch = a.nchunks;
  const int crank = (int)cluster_ctarank();
  const long long gpe = (a.t_end - a.t_begin + CL - 1) / CL;  // groups per ear (this launch's tiles)
  const long long ngroups = gpe * a.ears;
  const long long g0 = ngroups * cluster_id_x() / num_clusters_x();
  const long long g1 = ngroups * (cluster_id_x() + 1) / num_clusters_x();
  const long long u0 = g0 * nch, u1 = g1 * nch;
  const unsigned short cmask = (unsigned short)((1u << CL) - 1u);

  if (warp == 0) {
    // ===== G chunk producer =====
    if (elect_one()) {
      int bs = 0;
      unsigned bph = 0;
      const unsigned char* g = reinterpret_cast<const unsigned char*>(a.g);
      for (long long u = u0; u < u1; ++u) {
        const int c = (int)(u % nch);
        const int e = (int)(u / nch / gpe);
        PW(0, mbar_wait_sleep(&b_empty[bs], bph ^ 1u));  // the stage is free in every CTA of the cluster
        mbar_arrive_expect_tx(&b_full[bs], (unsigned)b_chunk_bytes);
        // this CTA loads one 16-byte-aligned slice of the chunk for the whole cluster
        const int sl0 = (int)((long long)b_chunk_bytes / 16 * crank / CL) * 16;
        const int sl1 = (int)((long long)b_chunk_bytes / 16 * (crank + 1) / CL) * 16;
        bulk_load_multicast(sB + bs * b_chunk_bytes + sl0, g + ((long long)e * nch + c) * b_chunk_bytes + sl0,
                            (unsigned)(sl1 - sl0), &b_full[bs], cmask);
        if (++bs == kMmaBStages) {
          bs = 0;
          bph ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(kMmaN >> 3) << 17) | ((uint32_t)(kMmaM >> 4) << 24);
      int bs = 0, as = 0, ab = -1, nit = -1;
      unsigned bph = 0, aph = 0, a_ph[2] = {0u, 0u};
      long long cur = -1;
      const unsigned sb = smem_u32(sB);
      for (long long u = u0; u < u1; ++u) {
        const long long item = u / nch;
        const int cu = (int)(u - item * nch);
        if (item != cur) {
          ++nit;
          if (ring) {
            PW(1, mbar_wait_sleep(&a_full[nit & 1], (unsigned)((nit >> 1) & 1)));  // hi rows of item nit
          } else {
            if (ab >= 0) mma_commit(&a_empty[ab]);  // this A buffer is free once its MMAs retire
            ab = (ab + 1) % NA;
            PW(1, mbar_wait_sleep(&a_full[ab], a_ph[ab]));
            a_ph[ab] ^= 1u;
          }
          cur = item;
        }
        PW(2, mbar_wait_sleep(&b_full[bs], bph));
        PW(3, mbar_wait_sleep(&acc_empty[as], aph ^ 1u));
        tmem_fence_after();
        const unsigned d = tbase + (unsigned)(as * kMmaN);
        const int hs = (2 * nit) % 3, ls = (2 * nit + 1) % 3;
        const unsigned at = tbase + (unsigned)(kMmaAccCols + (ring ? 0 : ab * KP));  // [hi | lo] KP/2 columns each
        const unsigned a_hi = ring ? at + (unsigned)(hs * (KP / 2)) : at;
        const unsigned a_lo = ring ? at + (unsigned)(ls * (KP / 2)) : at + (unsigned)(KP / 2);
        int acc = 0;
#pragma unroll 1
        for (int p = 0; p < 3; ++p) {  // hi*hi, hi*lo, lo*hi
          if (ring && p == 2) {
            if (cu == nch - 1) mma_commit(&slot_free[hs]);  // the item's hi rows are done
            if (cu == 0) PW(1, mbar_wait_sleep(&lo_full[nit & 1], (unsigned)((nit >> 1) & 1)));
          }
          const unsigned pa = p == 2 ? a_lo : a_hi;
          const unsigned pb = sb + (unsigned)(bs * b_chunk_bytes + (p == 1 ? 1 : 0) * b_part_bytes);
          for (int ks = 0; ks < KS; ++ks) {
#if !TOEP_MMA_NOMMA
            mma_f16_ts(d, pa + 8 * ks, mma_sdesc(pb + ks * kMmaN * 32), idesc, acc);
#endif
            acc = 1;
          }
        }
        if (ring && cu == nch - 1) mma_commit(&slot_free[ls]);  // and its lo rows
        mma_commit_multicast(&b_empty[bs], cmask);
        mma_commit(&acc_full[as]);
        if (++bs == kMmaBStages) {
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
    // ===== A builders: stage 1 + Hankel rows into TMEM =====
    const int bt = tid - 64;
    const int q = warp & 3;           // TMEM lane quarter
    const int sub = (warp - 2) >> 2;  // which columns of the row this warp writes
    const int YF = kMmaM + KP - 1;    // yf samples of an item
    const int YL = YF + a.lf_pad - 1; // y samples feeding them
    const int n8 = KP / 16;           // 8-column groups per part
    const int g0 = sub ? (n8 + 1) / 2 : 0, g1 = sub ? n8 : (n8 + 1) / 2;
    unsigned a_ph[2] = {0u, 0u};
    long long cur = -1;
    int cur_e = -1, nitem = 0;
    float chk = 0.f;
    for (long long u = u0; u < u1; ++u) {
      const long long item = u / nch;
      if (item == cur) continue;
      cur = item;
      const int ab = nitem % NA;
      const int e = (int)(item / gpe), ti = a.t_begin + (int)(item % gpe) * CL + crank;
      const long long T0 = (long long)ti * kMmaM;
      const long long y0 = T0 - (KP - 1) - (a.lf_pad - 1);
      if (e != cur_e)
        for (int i = bt; i < a.lf_pad; i += kMmaBuilders) s_f[i] = a.f[(long long)e * a.lf_pad + i];
      cur_e = e;
      float ymx = 0.f;
      for (int i = bt; i < YL; i += kMmaBuilders) {
        const long long t = y0 + i;
        const float v = (t >= 0 && t < a.nx) ? __ldg(a.x + t) : 0.f;
        chk = fmaf(v, 0.f, chk);
        ymx = fmaxf(ymx, fabsf(v));
        s_y[i] = v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ymx = fmaxf(ymx, __shfl_xor_sync(0xffffffffu, ymx, o));
      if (lane == 0) s_red[8 + warp - 2] = ymx;
      builders_sync();
      // a tile of tiny (e.g. fp32-subnormal) input is scaled up by 2^pexp before
      // the FIR, so stage 1 keeps full fp32 precision; pexp joins the tile exponent
      ymx = 0.f;
      for (int w = 0; w < kMmaBuilderWarps; ++w) ymx = fmaxf(ymx, s_red[8 + w]);
      const int pexp = (ymx > 0.f && ymx < 0x1p-64f) ? -ilogbf(ymx) : 0;
      if (pexp) {
        const float p1 = exp2i(pexp / 2), p2 = exp2i(pexp - pexp / 2);
        for (int i = bt; i < YL; i += kMmaBuilders) s_y[i] = s_y[i] * p1 * p2;
        builders_sync();
      }
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
      // max |yf| * 2^sexp in [2^13, 2^14); sexp in [-114, 162] (subnormal tiles
      // included), applied as two exact power-of-two factors so neither overflows
      const int sexp = mx > 0.f ? 13 - ilogbf(mx) : 0;
      const float sc1 = exp2i(sexp / 2), sc2 = exp2i(sexp - sexp / 2);
      if (bt == 0) {
        PW(5, mbar_wait_sleep(&sc_empty[nitem & 1], (unsigned)(((nitem >> 1) & 1) ^ 1)));
        s_sc[nitem & 1] = __int_as_float(sexp + pexp);
        mbar_arrive(&sc_full[nitem & 1]);
      }
      if (ring) {
        // hi rows into slot (2i) % 3, then lo rows into (2i+1) % 3, each once
        // the MMAs of its previous occupant have retired (use k of a slot
        // waits for completion k-1 of slot_free; a fresh barrier passes k = 0)
        const float* src = s_yf + (32 * q + lane + KP - 1);
#pragma unroll 1
        for (int part = 0; part < 2; ++part) {
          const int g = 2 * nitem + part, slot = g % 3, k = g / 3;
          PW(4, mbar_wait_sleep(&slot_free[slot], (unsigned)((k & 1) ^ 1)));
          tmem_fence_after();
          const unsigned ta = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(kMmaAccCols + slot * (KP / 2));
#pragma unroll 1
          for (int gi = g0; gi < g1; ++gi) {
            const int j0 = 8 * gi;
            unsigned w[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float x0 = src[-2 * (j0 + j)] * sc1 * sc2, x1 = src[-2 * (j0 + j) - 1] * sc1 * sc2;
              const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
              w[j] = part == 0 ? pack_half2(h0, h1)
                               : pack_half2(__float2half_rn(x0 - __half2float(h0)),
                                            __float2half_rn(x1 - __half2float(h1)));
            }
            tmem_st8(ta + j0, w);
          }
          tmem_wait_st();
          tmem_fence_before();
          builders_sync();
          if (bt == 0) mbar_arrive(part == 0 ? &a_full[nitem & 1] : &lo_full[nitem & 1]);
        }
        ++nitem;
        continue;
      }
      // the MMAs that last read this A buffer must have retired
      PW(4, mbar_wait_sleep(&a_empty[ab], a_ph[ab] ^ 1u));
      a_ph[ab] ^= 1u;
      tmem_fence_after();
      {
        // this lane's Hankel row: A[t][o] = yf[T0 + t - o], column j = {A[t][2j], A[t][2j+1]}
        const float* src = s_yf + (32 * q + lane + KP - 1);
        const unsigned ta = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(kMmaAccCols + ab * KP);
#pragma unroll 1
        for (int gi = g0; gi < g1; ++gi) {
          const int j0 = 8 * gi;
          unsigned hw[8], lw[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x0 = src[-2 * (j0 + j)] * sc1 * sc2, x1 = src[-2 * (j0 + j) - 1] * sc1 * sc2;
            const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
            hw[j] = pack_half2(h0, h1);
            lw[j] = pack_half2(__float2half_rn(x0 - __half2float(h0)), __float2half_rn(x1 - __half2float(h1)));
          }
          tmem_st8(ta + j0, hw);
          tmem_st8(ta + KP / 2 + j0, lw);
        }
        tmem_wait_st();
      }
      tmem_fence_before();
      builders_sync();
      if (bt == 0) mbar_arrive(&a_full[ab]);
      ++nitem;
    }
    if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
  } else {
    // ===== epilogue: TMEM -> registers -> shared staging -> TMA store =====
    const int ew = warp - 2 - kMmaBuilderWarps;
    const int q = warp & 3;    // TMEM lane quarter of this warp
    const int half = ew >> 2;  // which 64 of the chunk's 128 columns
    const int nstg = L.nstg;
    float* stg0 = reinterpret_cast<float*>(sm + L.st_off) + ew * nstg * 32 * 32;
    int sbuf = 0;
    const unsigned tq = tbase + ((unsigned)(32 * q) << 16);
    int as = 0;
    unsigned aph = 0;
    long long cur = -1;
    int nitem = -1;
    int tsexp = 0;
    float* fa = reinterpret_cast<float*>(sm + L.fac_off) + ew * 128;  // [2][64] factors of this warp's columns
    for (long long u = u0; u < u1; ++u) {
      const long long item = u / nch;
      const int c = (int)(u % nch);
      const int e = (int)(item / gpe), ti = a.t_begin + (int)(item % gpe) * CL + crank;
      if (item != cur) {
        if (nitem >= 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sc_empty[nitem & 1]);
        }
        ++nitem;
        mbar_wait_sleep(&sc_full[nitem & 1], (unsigned)((nitem >> 1) & 1));
        tsexp = __float_as_int(s_sc[nitem & 1]);
        cur = item;
      }
      // unscale = 2^-(tile exponent + G exponent): one factor per chunk, or per
      // column (direction) when the chunk's directions span more than 2^12 in
      // gain ("wide"); two factors whenever one would leave the normal range.
      // The chunk's exponents are loaded before the accumulator wait (their
      // latency hides behind it).
      const int* gx = a.gexp + ((long long)e * nch + c) * (kMmaN + 1);
      const int gwide = __ldg(gx + kMmaN), g0 = __ldg(gx);
      PW(6, mbar_wait_sleep(&acc_full[as], aph));
      tmem_fence_after();
      const long long t0 = (long long)ti * kMmaM + 32 * q;
      const bool wide = gwide != 0;
      float uc1 = 1.f, uc2 = 1.f;
      bool one = true;  // 2^-E is a normal float: one exact multiply
      if (!wide) {
        const int E = tsexp + g0;
        one = E >= -127 && E <= 126;
        uc1 = one ? exp2i(-E) : exp2i(-(E / 2));
        uc2 = exp2i(-(E - E / 2));
      } else {
        __syncwarp();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int E = tsexp + gx[64 * half + 32 * h2 + lane];
          fa[32 * h2 + lane] = exp2i(-(E / 2));
          fa[64 + 32 * h2 + lane] = exp2i(-(E - E / 2));
        }
        __syncwarp();
      }
      if (t0 < a.out_len && ti < a.t_end) {
#pragma unroll 1
        for (int blk = 0; blk < 2; ++blk) {
          const int col = 64 * half + 32 * blk;  // accumulator column = direction within the chunk
          const int d0 = c * kMmaN + col;
          if (d0 >= a.dirs) break;
          float* stg = stg0 + sbuf * 32 * 32;
          float vv[2][16];  // both 16-column loads in flight while the staging buffer frees up
          tmem_ld16(vv[0], tq + (unsigned)(as * kMmaN + col));
          tmem_ld16(vv[1], tq + (unsigned)(as * kMmaN + col + 16));
          if (lane == 0) {  // the store that last used this buffer has read it
            if (nstg == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          tmem_wait_ld();
#pragma unroll
          for (int cb = 0; cb < 32; cb += 16) {
            const float* v = vv[cb >> 4];
            if (!wide && one) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) stg[(cb + jj) * 32 + lane] = v[jj] * uc1;
            } else if (!wide) {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj) stg[(cb + jj) * 32 + lane] = v[jj] * uc1 * uc2;
            } else {
#pragma unroll
              for (int jj = 0; jj < 16; ++jj)
                stg[(cb + jj) * 32 + lane] = v[jj] * fa[32 * blk + cb + jj] * fa[64 + 32 * blk + cb + jj];
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (elect_one()) {
            tma_store_3d(&tm, stg, (int)t0, d0, e);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          if (++sbuf == nstg) sbuf = 0;
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
    if (lane == 0) bulk_wait_all();
  }
#if TOEP_MMA_PROF
  if (blockIdx.x == 7 && lane == 0 && (warp <= 2 || warp == 10))
    printf("prof cta7 warp %d total %lld: b_empty %lld a_full %lld b_full %lld acc_empty %lld a_empty %lld sc_empty %lld acc_full %lld\n",
           warp, clock64() - t_start, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5], prof[6]);
#endif
  tmem_fence_before();
  cluster_sync_all();  // no CTA leaves while cluster peers may still multicast into it
  if (warp == 0) tmem_dealloc<512>(tbase);
}

// G[e][c] chunk = [hi, lo][canonical 128 x kpad] fp16 of the dense rows of
// directions 128c .. 128c+127.  Rows are scaled by powers of two so that the
// largest |g| lands in [2^13, 2^14): one exponent for the whole chunk when its
// directions' maxima lie within 2^12 of each other (every row keeps the full
// hi/lo precision), else one per row ("wide" chunk; the epilogue unscales per
// column).  gexp[e][c] = {128 row exponents, wide flag}.  One block of kMmaN
// threads (one per direction row) per (ear, chunk).
__global__ void __launch_bounds__(kMmaN) k_build_gmma(const int2* __restrict__ raw, const int* __restrict__ nnz,
                                                     int dirs, int stride, int kpad, int nchunks,
                                                     __half* __restrict__ g, int* __restrict__ gexp) {
  __shared__ int s_lo[kMmaN / 32], s_hi[kMmaN / 32];
  const int c = blockIdx.x, e = blockIdx.y, r = threadIdx.x, d = c * kMmaN + r;
  const bool real = d < dirs;
  const int row = e * dirs + d;
  const int n = real ? nnz[row] : 0;
  const int2* taps = raw + (long long)row * stride;
  float mx = 0.f;
  for (int k = 0; k < n; ++k) mx = fmaxf(mx, fabsf(__int_as_float(taps[k].y)));
  // row exponent: 13 - ilogb(max); rows without taps do not constrain the chunk
  const int q = mx > 0.f ? 13 - ilogbf(mx) : 0;
  int lo = mx > 0.f ? q : INT_MAX, hi = mx > 0.f ? q : INT_MIN;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((r & 31) == 0) {
    s_lo[r >> 5] = lo;
    s_hi[r >> 5] = hi;
  }
  __syncthreads();
  lo = INT_MAX;
  hi = INT_MIN;
  for (int w = 0; w < kMmaN / 32; ++w) {
    lo = min(lo, s_lo[w]);
    hi = max(hi, s_hi[w]);
  }
  const bool wide = hi != INT_MIN && hi - lo > 12;
  const int qc = lo == INT_MAX ? 0 : lo;  // the loudest row's exponent
  const int qexp = wide ? (mx > 0.f ? q : qc) : qc;
  int* gx = gexp + ((long long)e * nchunks + c) * (kMmaN + 1);
  gx[r] = qexp;
  if (r == 0) gx[kMmaN] = wide ? 1 : 0;
  unsigned char* base = reinterpret_cast<unsigned char*>(g) + ((long long)e * nchunks + c) * 2 * kMmaN * kpad * 2;
  for (int k = 0; k < n; ++k) {  // taps are unique offsets; everything else stays zero (memset)
    const int o = taps[k].x;
    const float x = ldexpf(__int_as_float(taps[k].y), qexp);
    const __half h = __float2half_rn(x);
    const __half l = __float2half_rn(x - __half2float(h));
    *reinterpret_cast<__half*>(base + mma_canon(r, o, kMmaN)) = h;
    *reinterpret_cast<__half*>(base + kMmaN * kpad * 2 + mma_canon(r, o, kMmaN)) = l;
  }
}

int render_mma_kpad(int K) { return (K + 15) / 16 * 16; }
int render_mma_chunk() { return kMmaN; }

bool render_mma_supported(int K, int lf_pad) {
  const int kp = render_mma_kpad(K);
  if (kp > 256 || lf_pad > 512) return false;
  if (kMmaAccCols + kp > 512) return false;  // TMEM: accumulators + one A buffer (hi, lo)
  return mma_smem(kp, lf_pad).total <= 227 * 1024;
}

size_t render_mma_gbytes(int ears, int dirs, int K) {
  const int kp = render_mma_kpad(K);
  const int nch = (dirs + kMmaN - 1) / kMmaN;
  return (size_t)ears * nch * 2 * kMmaN * kp * 2;
}

size_t render_mma_gexp_ints(int ears, int dirs) {
  return (size_t)ears * ((dirs + kMmaN - 1) / kMmaN) * (kMmaN + 1);
}

cudaError_t build_render_mma_tables(const int2* raw, const int* nnz, int dirs, int ears, int stride, int K,
                                    void* g, int* gexp, cudaStream_t st) {
  const int kp = render_mma_kpad(K);
  const int nch = (dirs + kMmaN - 1) / kMmaN;
  cudaError_t e = cudaMemsetAsync(g, 0, render_mma_gbytes(ears, dirs, K), st);
  if (e != cudaSuccess) return e;
  k_build_gmma<<<dim3(nch, ears), kMmaN, 0, st>>>(raw, nnz, dirs, stride, kp, nch, reinterpret_cast<__half*>(g),
                                                 gexp);
  return cudaGetLastError();
}

template <int CL>
static void mma_cluster_cfg(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr, int smem) {
  cfg = {};
  cfg.blockDim = dim3(kMmaThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
}

template <int CL>
static cudaError_t launch_mma_cl(const RenderMmaArgs& a, const CUtensorMap& map, int grid, int smem, cudaStream_t st) {
  cudaError_t err = ensure_smem(reinterpret_cast<const void*>(k_render_mma<CL>), smem);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  mma_cluster_cfg<CL>(cfg, attr, smem);
  cfg.stream = st;
  cfg.gridDim = dim3((unsigned)grid);
  err = cudaLaunchKernelEx(&cfg, k_render_mma<CL>, a, map);
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

template <int CL>
static int max_clusters_for(int sm_count, int smem) {
  if (ensure_smem(reinterpret_cast<const void*>(k_render_mma<CL>), smem) != cudaSuccess) return 1;
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  mma_cluster_cfg<CL>(cfg, attr, smem);
  cfg.gridDim = dim3((unsigned)(std::max(1, sm_count / CL) * CL));
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k_render_mma<CL>, &cfg) != cudaSuccess || n < 1) n = std::max(1, sm_count / CL);
  cudaGetLastError();
  return n;
}

#ifndef TOEP_MMA_FILL
#define TOEP_MMA_FILL 1
#endif
#ifndef TOEP_MMA_FILL_RATE
#define TOEP_MMA_FILL_RATE 1.0
#endif
#ifndef TOEP_MMA_FILL_CL
#define TOEP_MMA_FILL_CL 2
#endif
constexpr int kMmaFillCluster = TOEP_MMA_FILL_CL;

// Kernel launches one launch_render_mma call makes for this many tiles (1, or
// 2 with the fill launch on the SMs the clusters leave idle).
int render_mma_launches(int n_titems, int kpad, int lf_pad, int sm_count) {
  const MmaSmem L = mma_smem(kpad, lf_pad);
  const int main_ctas = max_clusters_for<kMmaCluster>(sm_count, L.total) * kMmaCluster;
  const int fill = TOEP_MMA_FILL ? (sm_count - main_ctas) / kMmaFillCluster * kMmaFillCluster : 0;
  return (fill > 0 && n_titems >= 4 * sm_count) ? 2 : 1;
}

// Persistent launch: exactly the kMmaCluster-CTA clusters that can be
// co-resident (GPC sizes are not multiples of 6: 22 clusters cover 132 of a
// B200's 148 SMs), plus, concurrently on a side stream, small clusters on the
// SMs left over; each launch takes a share of every ear's tiles in proportion
// to its measured throughput.
cudaError_t launch_render_mma(const RenderMmaArgs& a, const CUtensorMap& map, const MmaFillStreams& fs,
                              int sm_count, cudaStream_t st) {
  const MmaSmem L = mma_smem(a.kpad, a.lf_pad);
  static std::mutex mu;
  static int clusters[64] = {};  // per device: co-resident kMmaCluster-CTA clusters
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  int ncl;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!clusters[dev]) {
      clusters[dev] = max_clusters_for<kMmaCluster>(sm_count, L.total);
      if (getenv("TOEP_VERBOSE"))
        fprintf(stderr, "k_render_mma: %d clusters of %d CTAs + fill on %d SMs\n", clusters[dev], kMmaCluster,
                sm_count);
    }
    ncl = clusters[dev];
  }
  const int main_ctas = ncl * kMmaCluster;
  const int fill = TOEP_MMA_FILL ? (sm_count - main_ctas) / kMmaFillCluster * kMmaFillCluster : 0;
  RenderMmaArgs m = a;
  m.t_begin = 0;
  m.t_end = a.n_titems;
  // the fill launch runs on the renderer's own side stream (fork/join events),
  // so distinct renderers never share a stream; without one, one launch
  if (fill <= 0 || a.n_titems < 4 * sm_count || !fs.side)
    return launch_mma_cl<kMmaCluster>(m, map, main_ctas, L.total, st);
  const double share = main_ctas / (main_ctas + TOEP_MMA_FILL_RATE * fill);
  const int split = std::min(a.n_titems, ((int)(a.n_titems * share) + kMmaCluster - 1) / kMmaCluster * kMmaCluster);
  m.t_end = split;
  RenderMmaArgs f = a;
  f.t_begin = split;
  f.t_end = a.n_titems;
  if ((err = cudaEventRecord(fs.fork, st)) != cudaSuccess) return err;
  if ((err = cudaStreamWaitEvent(fs.side, fs.fork, 0)) != cudaSuccess) return err;
  if ((err = launch_mma_cl<kMmaCluster>(m, map, main_ctas, L.total, st)) != cudaSuccess) return err;
  if ((err = launch_mma_cl<kMmaFillCluster>(f, map, fill, L.total, fs.side)) != cudaSuccess) return err;
  if ((err = cudaEventRecord(fs.join, fs.side)) != cudaSuccess) return err;
  return cudaStreamWaitEvent(st, fs.join, 0);
}

}  // namespace toep
