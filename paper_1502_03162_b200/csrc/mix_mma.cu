// Tensor-core mixdown (configs 4 offline and 5): the g-first partial mix
//   z_e[t] = sum_s (y_s * g_{e,dir(s)})[t]
// of many sources, each at one direction, as a GEMM on the tcgen05 tensor
// cores followed by an overlap-add.
//
// Reference semantics: the sum over sources of toepnmf's Renderer.render
// (pkg/src/toepnmf/engine/__init__.py:238-260 = conv_dense then conv_sparse,
// engine/_kernels.pyx:11-44), reordered reflection-first by the associativity
// the paper factorizes for (pkg/tests/test_acceptance.py:283-300);
// the resonance f_e is applied once to z afterwards (k_fir).
//
// Formulation.  Sources sharing a direction are summed first (Y_d = sum y_s).
// With n = (e, o) the output column for ear e and tap offset o,
//     W[t][n] = sum_d Y_d[t] * G[d][n],   G[d][(e,o)] = g_{e,d}[o]
//     z_e[t]  = sum_o W[t - o][(e,o)]                       (overlap-add)
// The first line is a dense GEMM with M = time, K = directions, N = ears x
// taps (2 x 104 = 208 at K = 100): the zero taps of the sparse g cost tensor
// work, which has headroom -- the kernel is bound by the one read of every
// source sample from HBM (4 B per source sample, 47 GB at config 5).  The
// W formulation needs no halo on the loads: a tile of 256 samples reads
// exactly samples [t0, t0+256) of each source; the (K-1)-sample tail of its
// overlap-add ("overhang") is kept per tile and added by k_mix_finish.
//
// fp32 accuracy from fp16 operands as in render_mma.cu: x = hi + lo,
// products hi*hi + hi*lo + lo*hi into fp32 TMEM accumulators.  G columns are
// normalised per direction by 2^gamma_d (host); the A value of row d is
// Y_d * 2^-gamma_d * 2^sexp (exact power-of-two scaling, undone in the
// epilogue).  The launch scale 2^sexp is fixed per mixer; every tile records
// max |Y_d 2^-gamma_d| and the main pass's last CTA lists the tiles whose values left the
// fp16-safe window (overflow, or so small that the low half loses bits while
// the tile still matters); a second launch of this kernel re-renders exactly
// those tiles with their own scale.  Results are a deterministic function of
// the input.
//
// Persistent CTA per SM (28 warps), tile = 256 samples = two 128-row blocks:
//   warps 0, 3  source producers (one thread each, alternate gathers): the
//               K-step's source rows, 4 per cp.async.bulk.tensor tile::gather4
//               (1 KB per row) into a ring of 1 KB slots; a K-step's rows
//               complete on one mbarrier (one gather4 occupies the TMA unit
//               ~90 cycles, so 4 KB per op keeps it ahead of HBM; the pattern
//               sustains ~7 TB/s, tools/microbench/gather_rate.cu)
//   warp 1      G producer: the K-step's G (hi, lo; canonical K-major
//               SWIZZLE_NONE, 13 KB at N = 208) into a 3-stage ring
//   warp 2      MMA issuer: per K-step 2 row blocks x 3 products of
//               tcgen05.mma M=128 N=208 K=16 (A from TMEM, G from smem)
//   warps 4-19  A builders (lane = time; 4 warps per lane quarter: row block x
//               half of the K-step's rows): sum each direction row's <= 4
//               source slices, scale, split hi/lo, tcgen05.st into a 3-slot
//               TMEM ring
//   warps 20-27 epilogue (row block x lane quarter): tcgen05.ld of W,
//               overlap-add through warp shuffles into per-lane registers,
//               combine of the 8 windows in shared memory, z stores + overhang
// The K-step tables (source rows, row info) are identical for every tile and
// sit in shared memory; the source ring takes the rest.
// TMEM: accumulators [0, 2N), A slots [416, 512) (32 columns each).
#include <algorithm>
#include <cstdio>
#include <cuda_fp16.h>

#include "common.cuh"
#include "launch.h"

namespace toep {

constexpr int kMxBuildWarps = 16;  // 4 per TMEM lane quarter: (row block, half of the K-step's 16 rows)
constexpr int kMxEpiWarps = 8;     // one per (row block, lane quarter)
constexpr int kMxWarps = 4 + kMxBuildWarps + kMxEpiWarps;
constexpr int kMxThreads = 32 * kMxWarps;
constexpr int kMxKR = 16;      // K-step barrier ring
#ifndef TOEP_MIX_GR
#define TOEP_MIX_GR 3
#endif
constexpr int kMxGR = TOEP_MIX_GR;  // G stages
constexpr int kMxAR = 3;       // A slots in TMEM (32 columns each: row block 0 hi, lo, row block 1 hi, lo)
constexpr int kMxACol = 416;   // first A-slot column (accumulators: 2 row blocks x N <= 416)
constexpr int kMxSlotBytes = kMixTile * 4;
constexpr int kMxWindows = 8;  // overlap-add windows per tile: (row block, lane quarter)
constexpr int kMxGroupKs = 96; // K-steps accumulated in TMEM before a drain (bounds the accumulation error)

__device__ __forceinline__ uint64_t mx_sdesc(unsigned saddr) {
  // canonical K-major, SWIZZLE_NONE: LBO (K halves) 128 B, SBO (8-row groups) 256 B, version 1
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mx_mma(unsigned d_tmem, unsigned a_tmem, uint64_t db, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mx_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mx_st4(unsigned ta, unsigned a0, unsigned a1, unsigned a2, unsigned a3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(a0), "r"(a1), "r"(a2),
               "r"(a3)
               : "memory");
}
// four source rows (tensor-map rows r0..r3, columns [col, col + 256)) -> 4 consecutive 1 KB slots
__device__ __forceinline__ void mx_gather4(void* sdst, const CUtensorMap* tm, int col, int4 r, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(smem_u32(sdst)),
      "l"(tm), "r"(col), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ unsigned mx_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);  // a -> low half (column element 2j), b -> high half
  return *reinterpret_cast<const unsigned*>(&h);
}
__device__ __forceinline__ float p2f(int e) { return __int_as_float((127 + e) << 23); }  // 2^e, e in [-126, 127]

// the direction sums of 8 rows of C slices each: slot (C r + k) of the row
// block, compile-time offsets (all 8 C loads issue before the adds)
template <int C>
__device__ __forceinline__ void mx_row_sums(const float* __restrict__ base, float (&v)[8]) {
  float L[8 * C];
#pragma unroll
  for (int i = 0; i < 8 * C; ++i) L[i] = base[i * kMixTile];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if constexpr (C == 4) v[r] = (L[4 * r] + L[4 * r + 2]) + (L[4 * r + 1] + L[4 * r + 3]);
    else if constexpr (C == 3) v[r] = (L[3 * r] + L[3 * r + 2]) + L[3 * r + 1];
    else if constexpr (C == 2) v[r] = L[2 * r] + L[2 * r + 1];
    else v[r] = L[r];
  }
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct MxSmem {
  int ring, g, ebuf, src, rows, rowf, ksn, misc, bars, total;
};
// Shared-memory layout; the source ring takes what the tables leave of the
// 227 KB (ring = 0 asks for the ring size that fits, >= kMxMinRing slots).
constexpr int kMxSmemMax = 227 * 1024 - 1024;  // static shared memory + slack
constexpr int kMxMinRing = 2 * kMixKsSrcs;      // 1 KB slots (two full K-steps)
__host__ __device__ inline MxSmem mx_smem(int N, int ears, int nr, int nsrc4, int KS, int ring) {
  MxSmem L{};
  int off = 0;
  L.g = off;  // [kMxGR][hi, lo][N x 16] fp16
  off += kMxGR * N * 64;
  L.ebuf = off;  // [kMxWindows][ears][32 * nr] fp32
  off += kMxWindows * ears * 32 * nr * 4;
  L.src = off;  // [nsrc4] source rows of the K-steps (uint16, 8-byte aligned groups of 4)
  off += ((nsrc4 + 7) & ~7) * 2;
  L.rows = off;  // [KS][16] row info
  off += KS * 64;
  L.rowf = off;  // [KS][16] main-pass row multipliers 2^(sexp - gamma_d)
  off += KS * 64;
  L.ksn = off;  // [KS] int2 {src offset, count}
  off += ((KS + 1) & ~1) * 8;
  L.misc = off;  // builder max per warp [16]
  off += 64;
  L.bars = off;
  off += (2 * kMxKR + 2 * kMxGR + 2 * kMxAR + 2) * 8;
  off = (off + 127) & ~127;
  L.ring = off;
  if (ring <= 0) ring = (kMxSmemMax - off) / kMxSlotBytes;
  off += ring * kMxSlotBytes;
  L.total = off;
  return L;
}

// tile sequence of this CTA: a contiguous range (main pass) or its share of
// the bad-tile list (fixup pass)
// Work units are (tile, K-step group): a tile whose K-steps exceed
// kMxGroupKs is accumulated in groups, each drained into z (the first group
// stores, later ones add) -- the tensor core's fp32 accumulation error grows
// with the accumulation count, so this bounds it for any source count.
struct MxTiles {
  const int* list;
  int j0, j1, cnt, ng;
  __device__ int tile_of(int t) const {
    if (!list) return j0 + t < j1 ? j0 + t : -1;
    const int k = t * (int)gridDim.x + (int)blockIdx.x;
    return k < cnt ? list[k] : -1;
  }
  __device__ int at(int i) const { return tile_of(i / ng); }  // unit i -> tile (-1: done)
  __device__ int group(int i) const { return i % ng; }
};

// tile scale exponent: the launch's in the main pass; in the fixup pass the
// one that puts the tile's recorded max |A| (at the launch scale) into
// [2^13, 2^14) -- integer arithmetic, so no intermediate under/overflows
__device__ __forceinline__ int mx_tile_sexp(const MixMmaArgs& a, int j) {
  if (!a.bad_list) return a.sexp;
  const float m = a.tile_max[j];
  return m > 0.f ? a.sexp + 13 - ilogbf(m) : a.sexp;
}
// tiles the fixup pass re-renders: max |A| at the launch scale outside the
// fp16-safe window [2^-3, 2^15] -- the hi half would overflow, or the lo half
// of the tile's largest values would not be a normal fp16 number; all-zero
// tiles are exact at any scale; non-finite input is reported by the z check
__device__ __forceinline__ bool mx_tile_bad(float s) {
  return isfinite(s) && s != 0.f && (s > 32768.f || s < 0.125f);
}
// 2^e for any e: two exact factors (each clamped to the normal range, where
// the value they scale would under/overflow anyway)
__device__ __forceinline__ float2 p2f2(int e) {
  const int e1 = max(-126, min(127, e >> 1)), e2 = max(-126, min(127, e - (e >> 1)));
  return make_float2(p2f(e1), p2f(e2));
}

#ifndef TOEP_MIX_PROF
#define TOEP_MIX_PROF 0
#endif
#ifndef TOEP_MIX_PRODUCTS
#define TOEP_MIX_PRODUCTS 3
#endif
// builders poll their barriers (short waits on the critical path); every
// other role suspends in try_wait (a polling warp steals issue slots from the
// builders: 8 spinning epilogue warps were ~20% of all issued instructions)
#if defined(TOEP_MIX_SLEEPALL) && TOEP_MIX_SLEEPALL
#define MX_BWAIT mbar_wait_sleep
#else
#define MX_BWAIT mbar_wait
#endif
#if TOEP_MIX_PROF
#define PROF_WAIT(slot, ...)         \
  do {                               \
    const long long _t0 = clock64(); \
    __VA_ARGS__;                     \
    prof[slot] += clock64() - _t0;   \
  } while (0)
#else
#define PROF_WAIT(slot, ...) __VA_ARGS__
#endif
#if !TOEP_MIX_PROF
#define PROF_MARK(slot) \
  do {                  \
  } while (0)
#endif

template <int CH, int NR>
__global__ void __launch_bounds__(kMxThreads, 1) k_mix_mma(MixMmaArgs a, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  const int N = a.N;
  const MxSmem L = mx_smem(N, a.ears, NR, a.nsrc4, a.KS, a.ring);
  const int RING = a.ring;
  const int gbytes = N * 64;
  float* ring = reinterpret_cast<float*>(sm + L.ring);
  unsigned char* sG = sm + L.g;
  float* ebuf = reinterpret_cast<float*>(sm + L.ebuf);
  float* s_bmax = reinterpret_cast<float*>(sm + L.misc);
  uint2* s_src4 = reinterpret_cast<uint2*>(sm + L.src);  // 4 x uint16 per gather
  int4* s_rows4 = reinterpret_cast<int4*>(sm + L.rows);
  float4* s_rowf4 = reinterpret_cast<float4*>(sm + L.rowf);
  int2* s_ksn = reinterpret_cast<int2*>(sm + L.ksn);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
  uint64_t* src_full = bars;
  uint64_t* src_empty = src_full + kMxKR;
  uint64_t* g_full = src_empty + kMxKR;
  uint64_t* g_empty = g_full + kMxGR;
  uint64_t* a_full = g_empty + kMxGR;
  uint64_t* a_empty = a_full + kMxAR;
  uint64_t* acc_full = a_empty + kMxAR;
  uint64_t* acc_empty = acc_full + 1;
  __shared__ unsigned s_tbase;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if TOEP_MIX_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long _tp = 0;
#define PROF_MARK(slot)                      \
  do {                                       \
    const long long _n = clock64();          \
    prof[slot] += _n - _tp;                  \
    _tp = _n;                                \
  } while (0)
  const long long t_start = clock64();
#endif

  if (warp == 3) tmem_alloc<512>(&s_tbase);
  if (tid == 0) {
    for (int i = 0; i < kMxKR; ++i) {
      mbar_init(&src_full[i], 1);
      mbar_init(&src_empty[i], kMxBuildWarps);
    }
    for (int i = 0; i < kMxGR; ++i) {
      mbar_init(&g_full[i], 1);
      mbar_init(&g_empty[i], 1);
    }
    for (int i = 0; i < kMxAR; ++i) {
      mbar_init(&a_full[i], kMxBuildWarps);
      mbar_init(&a_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kMxEpiWarps);
    mbar_fence_init();
  }
  // the K-step tables (identical for every tile) -> shared memory
  for (int i = tid; i < (a.nsrc4 >> 2); i += kMxThreads) s_src4[i] = __ldg(reinterpret_cast<const uint2*>(a.src) + i);
  for (int i = tid; i < a.KS * 4; i += kMxThreads) {
    s_rows4[i] = __ldg(reinterpret_cast<const int4*>(a.rows) + i);
    s_rowf4[i] = __ldg(reinterpret_cast<const float4*>(a.rowf) + i);
  }
  for (int i = tid; i < a.KS; i += kMxThreads) s_ksn[i] = __ldg(a.ks + i);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tbase = s_tbase;

  MxTiles tiles;
  tiles.list = a.bad_list;
  tiles.j0 = (int)((long long)a.n_tiles * blockIdx.x / gridDim.x);
  tiles.j1 = (int)((long long)a.n_tiles * (blockIdx.x + 1) / gridDim.x);
  tiles.cnt = a.bad_list ? *a.bad_count : 0;
  tiles.ng = (a.KS + kMxGroupKs - 1) / kMxGroupKs;
  const int KS = a.KS;
  const int KSG = (KS + tiles.ng - 1) / tiles.ng;  // K-steps per group

  if (warp == 0 || warp == 3) {
    // ===== source producers (one thread each in warps 0 and 3, on different SM
    //       sub-partitions): the K-step's source rows, 4 per tile::gather4,
    //       alternate gathers per thread (one gather4 costs ~100 issue cycles);
    //       both track the ring identically, warp 0 posts the expected bytes =====
    const int pid = warp == 0 ? 0 : 1;
    if (elect_one()) {
      long long seq = 0, fseq = 0;  // K-steps issued / released
      int pos = 0;                  // next free slot (a K-step never wraps: its slots restart at 0)
      int held = 0;                 // slots held by unreleased K-steps (incl. skipped tails)
      int hold[kMxKR];              // slots each in-flight K-step holds
      for (int i = 0;; ++i) {
        const int j = tiles.at(i);
        if (j < 0) break;
        const int col = j * kMixTile;
        const int kg0 = tiles.group(i) * KSG, kg1 = min(KS, kg0 + KSG);
        for (int ks = kg0; ks < kg1; ++ks) {
          const int2 info = s_ksn[ks];
          const int n = info.y & 0xffff;  // slots, a multiple of 8
          const int skip = pos + n > RING ? RING - pos : 0;
          while (seq - fseq >= kMxKR || held + skip + n > RING) {
            PROF_WAIT(0, mbar_wait_sleep(&src_empty[fseq % kMxKR], (unsigned)((fseq / kMxKR) & 1)));
            held -= hold[fseq % kMxKR];
            ++fseq;
          }
          if (pos + n > RING) pos = 0;
          hold[seq % kMxKR] = skip + n;
          held += skip + n;
          uint64_t* bar = &src_full[seq % kMxKR];
          if (pid == 0) mbar_arrive_expect_tx(bar, (unsigned)(n * kMxSlotBytes));
          const uint2* sl = s_src4 + (info.x >> 2);
          float* dst = ring + pos * kMixTile;
#pragma unroll 4
          for (int g = pid; g < (n >> 2); g += 2) {
            const uint2 r2 = sl[g];
            const int4 r = make_int4((int)(r2.x & 0xffffu), (int)(r2.x >> 16), (int)(r2.y & 0xffffu), (int)(r2.y >> 16));
            mx_gather4(dst + 4 * g * kMixTile, &tm, col, r, bar);
          }
          pos += n;
          ++seq;
        }
      }
    }
  } else if (warp == 1) {
    // ===== G producer =====
    if (elect_one()) {
      int gs = 0;
      unsigned gph = 0;
      for (int i = 0;; ++i) {
        if (tiles.at(i) < 0) break;
        const int kg0 = tiles.group(i) * KSG, kg1 = min(KS, kg0 + KSG);
        for (int ks = kg0; ks < kg1; ++ks) {
          PROF_WAIT(0, mbar_wait_sleep(&g_empty[gs], gph ^ 1u));
          mbar_arrive_expect_tx(&g_full[gs], (unsigned)gbytes);
          bulk_load(sG + gs * gbytes, a.g + (long long)ks * gbytes, (unsigned)gbytes, &g_full[gs]);
          if (++gs == kMxGR) {
            gs = 0;
            gph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 2) {
    // ===== MMA issuer: per K-step 2 row blocks x 3 products =====
    if (elect_one()) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const unsigned sg = smem_u32(sG);
      int gs = 0, as = 0;
      unsigned gph = 0, aph = 0, cph = 0;
      for (int i = 0;; ++i) {
        if (tiles.at(i) < 0) break;
        PROF_WAIT(2, mbar_wait_sleep(acc_empty, cph ^ 1u));  // the epilogue has drained the accumulators
        cph ^= 1u;
        tmem_fence_after();
        const int kg0 = tiles.group(i) * KSG, kg1 = min(KS, kg0 + KSG);
        for (int ks = kg0; ks < kg1; ++ks) {
          PROF_WAIT(0, mbar_wait_sleep(&g_full[gs], gph));
          PROF_WAIT(1, mbar_wait_sleep(&a_full[as], aph));
          tmem_fence_after();
          const unsigned bh = sg + (unsigned)(gs * gbytes), bl = bh + (unsigned)(N * 32);
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const unsigned d = tbase + (unsigned)(rb * N);
            const unsigned ah = tbase + (unsigned)(kMxACol + 32 * as + 16 * rb), al = ah + 8;
            mx_mma(d, ah, mx_sdesc(bh), idesc, ks > kg0);
#if TOEP_MIX_PRODUCTS > 1  // experiment knob: 3 products are needed for fp32 accuracy
            mx_mma(d, ah, mx_sdesc(bl), idesc, 1);
#endif
#if TOEP_MIX_PRODUCTS > 2
            mx_mma(d, al, mx_sdesc(bh), idesc, 1);
#endif
          }
          mx_commit(&a_empty[as]);
          mx_commit(&g_empty[gs]);
          if (++gs == kMxGR) {
            gs = 0;
            gph ^= 1u;
          }
          if (++as == kMxAR) {
            as = 0;
            aph ^= 1u;
          }
        }
        mx_commit(acc_full);
      }
    }
  } else if (warp >= 4 && warp < 4 + kMxBuildWarps) {
    // ===== A builders: lane = time; 8 of the K-step's 16 direction rows (<= 4 slices each) =====
    const int bw = warp - 4;
    const int q = warp & 3, rb = (bw >> 2) & 1, half = bw >> 3;
    const int tt = 128 * rb + 32 * q + lane;  // time within the tile
    const unsigned ta0 = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(kMxACol + 16 * rb + 4 * half);
    long long seq = 0;
    int pos = 0, as = 0;
    unsigned aph = 0;
    const bool fixup = a.bad_list != nullptr;
    float amax = 0.f;
#if TOEP_MIX_PROF
    _tp = clock64();
#endif
    for (int i = 0;; ++i) {
      const int j = tiles.at(i);
      if (j < 0) break;
      const int sexp = mx_tile_sexp(a, j);  // (samples past T arrive as zeros: TMA out-of-bounds fill)
      const int grp = tiles.group(i);
      if (grp == 0) amax = 0.f;
      const int kg0 = grp * KSG, kg1 = min(KS, kg0 + KSG);
      for (int ks = kg0; ks < kg1; ++ks) {
        const int ksy = s_ksn[ks].y;  // n | c0 << 16: 8 rows x c0 slots, then 8 rows x c1 (c = sources per row)
        const int n = ksy & 0xffff, c0 = ksy >> 16;
        // this warp's 8 row multipliers, read before the data wait (main pass)
        float4 m0 = make_float4(0.f, 0.f, 0.f, 0.f), m1 = m0;
        if (!fixup) {
          m0 = s_rowf4[4 * ks + 2 * half];
          m1 = s_rowf4[4 * ks + 2 * half + 1];
        }
        if (pos + n > RING) pos = 0;
        PROF_MARK(3);
        PROF_WAIT(0, MX_BWAIT(&src_full[seq % kMxKR], (unsigned)((seq / kMxKR) & 1)));
        PROF_MARK(7);
        float v[8];
        {
          const int c = half ? (n >> 3) - c0 : c0;  // this warp's half: one size class
          const float* base = ring + (pos + 8 * c0 * half) * kMixTile + tt;  // this warp's first row
          switch (c) {
            case 4: mx_row_sums<4>(base, v); break;
            case 3: mx_row_sums<3>(base, v); break;
            case 2: mx_row_sums<2>(base, v); break;
            default: mx_row_sums<1>(base, v); break;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&src_empty[seq % kMxKR]);
        PROF_MARK(4);
        unsigned hw[4], lw[4];
        float mul[8];
        if (!fixup) {  // 2^(sexp - gamma_d), precomputed
          mul[0] = m0.x; mul[1] = m0.y; mul[2] = m0.z; mul[3] = m0.w;
          mul[4] = m1.x; mul[5] = m1.y; mul[6] = m1.z; mul[7] = m1.w;
        } else {  // the tile's own exponent: two exact factors per row
          const int4 ra = s_rows4[4 * ks + 2 * half], rbv = s_rows4[4 * ks + 2 * half + 1];  // this warp's 8 rows
          const int ri[8] = {ra.x, ra.y, ra.z, ra.w, rbv.x, rbv.y, rbv.z, rbv.w};
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const float2 f = p2f2(sexp - (((ri[r] >> 9) & 0xff) - 128));
            v[r] *= f.x;
            mul[r] = f.y;
          }
        }
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
          const float x0 = v[r] * mul[r], x1 = v[r + 1] * mul[r + 1];
          amax = fmaxf(amax, fmaxf(fabsf(x0), fabsf(x1)));
          const unsigned h = mx_h2(x0, x1);
          const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
          hw[r / 2] = h;
          lw[r / 2] = mx_h2(x0 - hf.x, x1 - hf.y);
        }
        PROF_MARK(5);
        PROF_WAIT(1, MX_BWAIT(&a_empty[as], aph ^ 1u));
        PROF_MARK(7);
        tmem_fence_after();
        const unsigned ta = ta0 + (unsigned)(32 * as);
        mx_st4(ta, hw[0], hw[1], hw[2], hw[3]);
        mx_st4(ta + 8, lw[0], lw[1], lw[2], lw[3]);
        tmem_wait_st();
        tmem_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
        PROF_MARK(6);
        if (++as == kMxAR) {
          as = 0;
          aph ^= 1u;
        }
        pos += n;
        ++seq;
      }
      if (!a.bad_list && grp == tiles.ng - 1) {  // tile max (at the launch scale) for the fixup scan
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if (lane == 0) s_bmax[bw] = amax;
        named_sync(1, 32 * kMxBuildWarps);
        if (bw == 0 && lane == 0) {
          float m = 0.f;
          for (int w = 0; w < kMxBuildWarps; ++w) m = fmaxf(m, s_bmax[w]);
          a.tile_max[j] = m;
          __threadfence();  // before this CTA's arrival at the end (the last CTA scans the maxima)
        }
        named_sync(1, 32 * kMxBuildWarps);
      }
    }
  } else if (warp >= 4 + kMxBuildWarps) {
    // ===== epilogue: W -> overlap-add -> z (one warp per row block x lane quarter) =====
    const int ew = warp - 4 - kMxBuildWarps;
    const int q = warp & 3, rb = ew >> 2;
    const unsigned tq = tbase + ((unsigned)(32 * q) << 16) + (unsigned)(rb * N);
    const int ears = a.ears, K = a.K, KP = a.KP;
    const int win = 32 * NR;
    unsigned cph = 0;
    for (int i = 0;; ++i) {
      const int j = tiles.at(i);
      if (j < 0) break;
      float* eb = ebuf;
      float R0[NR], R1[NR];
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        R0[k] = 0.f;
        R1[k] = 0.f;
      }
      PROF_WAIT(0, mbar_wait_sleep(acc_full, cph));
      cph ^= 1u;
      tmem_fence_after();
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float w0[16], w1[16];
        tmem_ld16(w0, tq + (unsigned)(16 * c));
        if (ears > 1) tmem_ld16(w1, tq + (unsigned)(KP + 16 * c));
        tmem_wait_ld();
        if (c == CH - 1) {  // every accumulator column this warp reads has been read
          tmem_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
        }
        // W[t][o] (lane t) belongs to window position t + o: lane L collects
        // the positions = L (mod 32) from lane (L - o) mod 32
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int o = 16 * c + jj;
          if (o < K) {
            const int srcl = (lane - o) & 31;
            const float x0 = __shfl_sync(0xffffffffu, w0[jj], srcl);
            const float x1 = ears > 1 ? __shfl_sync(0xffffffffu, w1[jj], srcl) : 0.f;
            const int kb = o >> 5;
            if (srcl + (o & 31) < 32) {
              R0[kb] += x0;
              R1[kb] += x1;
            } else if (kb + 1 < NR) {
              R0[kb + 1] += x0;
              R1[kb + 1] += x1;
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        eb[(ew * ears) * win + 32 * k + lane] = R0[k];
        if (ears > 1) eb[(ew * ears + 1) * win + 32 * k + lane] = R1[k];
      }
      named_sync(2, 32 * kMxEpiWarps);
      // combine the 8 windows (fixed order): position P of the tile's 256 + K - 1
      const long long t0 = (long long)j * kMixTile;
      const bool grp0 = tiles.group(i) == 0;
      const float2 inv = p2f2(-mx_tile_sexp(a, j));
      const int npos = kMixTile + K - 1;
      const int et = tid - 32 * (4 + kMxBuildWarps);
      for (int idx = et; idx < ears * npos; idx += 32 * kMxEpiWarps) {
        const int e = idx / npos, P = idx - e * npos;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < kMxWindows; ++w) {
          const int b = 128 * (w >> 2) + 32 * (w & 3);
          if (P >= b && P < b + win) acc += eb[(w * ears + e) * win + (P - b)];
        }
        acc = acc * inv.x * inv.y;
        // the first K-step group of a tile stores, later groups add (same
        // thread, same position: program order)
        if (P < kMixTile) {
          if (t0 + P < a.zlen) {
            float* zp = a.z + (long long)e * a.z_pitch + t0 + P;
            *zp = grp0 ? acc : *zp + acc;
          }
        } else {
          float* op = a.ovh + ((long long)j * ears + e) * a.ovh_pitch + (P - kMixTile);
          *op = grp0 ? acc : *op + acc;
        }
      }
      named_sync(2, 32 * kMxEpiWarps);  // the windows are rewritten for the next tile
    }
  }
#if TOEP_MIX_PROF
  if (blockIdx.x == 0 && (warp <= 3 || warp == 4 || warp == 4 + kMxBuildWarps) &&
      (lane == 0 || prof[0] + prof[1] + prof[2] > 0) && (warp != 0 || lane == 0))
    printf("mixprof warp %d total %lld waits: %lld %lld %lld phases: top %lld loads %lld conv %lld st %lld\n", warp,
           clock64() - t_start, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5], prof[6]);
#endif
  tmem_fence_before();
  __syncthreads();
  if (warp == 3) tmem_dealloc<512>(tbase);
  if (a.scan_count) {  // main pass: the last CTA to finish lists the fixup pass's tiles
    __shared__ int s_last, s_n;
    if (tid == 0) {
      __threadfence();  // this CTA's tile maxima before its arrival
      s_last = atomicAdd(a.scan_done, 1u) == gridDim.x - 1;
      s_n = 0;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int j = tid; j < a.n_tiles; j += kMxThreads)
        if (mx_tile_bad(a.tile_max[j])) a.scan_list[atomicAdd(&s_n, 1)] = j;
      __syncthreads();
      if (tid == 0) {
        *a.scan_count = s_n;
        *a.scan_done = 0u;  // ready for the next call
      }
    }
  }
}

// Finish of the partial, one pass over z: the per-tile overhangs (the K - 1
// samples past each tile's end) are added at the next tile's start,
// z[e][256 (j+1) + p] += ovh[j][e][p] (the last tile's overhang is stored),
// and -- when `nonfinite` is set -- every finished sample is checked: the
// fused input check of the tensor mixdown (the reference's DataError for
// non-finite samples, engine/__init__.py:162-165).  A non-finite source sample
// makes its tile's z non-finite (sums, fp16 halves and products propagate
// inf/NaN), so the finished z is checked instead of every source sample
// (23 MB instead of 47 GB at config 5).
__global__ void __launch_bounds__(256) k_mix_finish(float* __restrict__ z, long long z_pitch, long long zlen,
                                                    const float* __restrict__ ovh, int ovh_pitch, int n_tiles,
                                                    int ears, int nov, int* __restrict__ nonfinite) {
  bool bad = false;
  for (int e = 0; e < ears; ++e) {
    float* ze = z + (long long)e * z_pitch;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < zlen;
         t += (long long)gridDim.x * blockDim.x) {
      const long long j = t / kMixTile - 1;  // the tile whose overhang reaches t
      const int p = (int)(t - (j + 1) * kMixTile);
      float v;
      if (j >= 0 && p < nov && j < n_tiles) {
        const float o = ovh[(j * ears + e) * ovh_pitch + p];
        v = (j + 1 < n_tiles ? ze[t] : 0.f) + o;
        ze[t] = v;
      } else {
        if (!nonfinite) continue;
        v = ze[t];
      }
      bad |= !isfinite(v);
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

int mix_mma_nr(int K) { return (32 + K - 1 + 31) / 32; }

// ring slots left by the tables (0 if the tables do not leave kMxMinRing slots)
int mix_mma_ring(int N, int ears, int K, int nsrc4, int KS) {
  const int nr = mix_mma_nr(K) <= 5 ? 5 : 8;
  const int ring = (kMxSmemMax - mx_smem(N, ears, nr, nsrc4, KS, 1).ring) / kMxSlotBytes;
  return ring >= kMxMinRing ? ring : 0;
}

template <int CH, int NR>
static cudaError_t launch_mix_mma_t(const MixMmaArgs& a, const CUtensorMap& tm, int grid, cudaStream_t st) {
  const int bytes = mx_smem(a.N, a.ears, NR, a.nsrc4, a.KS, a.ring).total;
  auto kern = k_mix_mma<CH, NR>;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), bytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kMxThreads, bytes, st>>>(a, tm);
  return cudaGetLastError();
}

cudaError_t launch_mix_mma(const MixMmaArgs& a_in, const CUtensorMap& tm, int* bad_list, int* bad_count,
                           int sm_count, cudaStream_t st) {
  if (a_in.N < 16 || a_in.N > 208 || a_in.N % 16 || a_in.K < 1) return cudaErrorInvalidValue;
  const int nr = mix_mma_nr(a_in.K);
  const int ch = (a_in.K + 15) / 16;
  MixMmaArgs a = a_in;
  a.bad_list = nullptr;
  a.bad_count = nullptr;
  a.scan_list = bad_list;  // the main pass's last CTA writes the fixup list
  a.scan_count = bad_count;
  a.scan_done = reinterpret_cast<unsigned*>(bad_count + 1);
  const int grid = std::max(1, std::min(sm_count, a.n_tiles));
  auto go = [&](const MixMmaArgs& x) -> cudaError_t {
    if (ch <= 7 && nr <= 5) return launch_mix_mma_t<7, 5>(x, tm, grid, st);
    if (ch <= 13 && nr <= 8) return launch_mix_mma_t<13, 8>(x, tm, grid, st);
    return cudaErrorInvalidValue;
  };
  cudaError_t e = go(a);
  if (e != cudaSuccess) return e;
  MixMmaArgs f = a;
  f.bad_list = bad_list;
  f.bad_count = bad_count;
  f.scan_list = nullptr;
  f.scan_count = nullptr;
  e = go(f);
  if (e != cudaSuccess) return e;
  const int nov = a.K - 1;
  if (nov > 0 || a.nonfinite) {
    const int blocks = (int)std::min<long long>((a.zlen + 255) / 256, (long long)sm_count * 8);
    k_mix_finish<<<std::max(blocks, 1), 256, 0, st>>>(a.z, a.z_pitch, a.zlen, a.ovh, a.ovh_pitch, a.n_tiles, a.ears,
                                                       nov, a.nonfinite);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace toep
