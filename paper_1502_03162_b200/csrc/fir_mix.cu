// Dense FIR, generic sparse fallback, g-first source mixdown and the streaming
// block step.
//
// Reference semantics:
//   dense FIR       <- conv_dense   (pkg/src/toepnmf/engine/_kernels.pyx:11-25)
//   sparse fallback <- conv_sparse  (pkg/src/toepnmf/engine/_kernels.pyx:28-44)
//   mixdown         <- sum over sources of Renderer.render (engine/__init__.py:238-260),
//                      reordered with the associativity the paper relies on
//                      (tests/test_acceptance.py:283-300):
//                      sum_s (y_s*f_e)*g_s,e = f_e * sum_s (y_s*g_s,e)
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace toep {

// ------------------------------------------------------------ dense FIR ----
constexpr int kFirChunk = 512;  // taps staged in shared memory per pass

__global__ void __launch_bounds__(kThreads) k_fir(FirArgs a) {
  __shared__ __align__(16) float s_x[padded_len(kW + kFirChunk)];
  __shared__ __align__(16) float s_h[kFirChunk];
  const int tid = threadIdx.x;
  const int c = blockIdx.y;
  const long long T0 = (long long)blockIdx.x * kW;
  const float* x = a.x + (long long)c * a.x_pitch;
  const float* h = a.h + (long long)c * a.h_pitch;
  float acc[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[r] = 0.f;
  for (int j0 = 0; j0 < a.nh_pad; j0 += kFirChunk) {
    const int nch = min(kFirChunk, a.nh_pad - j0);
    __syncthreads();
    for (int i = tid; i < nch; i += kThreads) s_h[i] = h[j0 + i];
    // s_x[k] = x[T0 - j0 - nch + k], k in [0, kW + nch)
    const long long xs = T0 - j0 - nch;
    for (int i = tid; i < kW + nch; i += kThreads) {
      const long long t = xs + i;
      s_x[padi(i)] = (t >= 0 && t < a.nx) ? __ldg(x + t) : 0.f;
    }
    __syncthreads();
    fir16_block(acc, s_x, nch + 16 * tid, s_h, nch);
  }
  __syncthreads();
  // stage through shared memory for coalesced row stores
  float* s_o = s_x;
#pragma unroll
  for (int r = 0; r < 16; ++r) s_o[padi(16 * tid + r)] = acc[r];
  __syncthreads();
  float* o = a.out + (long long)c * a.out_pitch;
  for (int i = tid; i < kW; i += kThreads) {
    const long long t = T0 + i;
    if (t < a.out_len) o[t] = s_o[padi(i)];
  }
}

cudaError_t launch_fir(const FirArgs& a, cudaStream_t st) {
  if (a.out_len <= 0 || a.channels <= 0) return cudaSuccess;
  const long long tiles = (a.out_len + kW - 1) / kW;
  dim3 grid((unsigned)tiles, (unsigned)a.channels);
  k_fir<<<grid, kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------- generic sparse (any length) ----
constexpr int kBand = 1024;

__global__ void __launch_bounds__(kThreads) k_sparse_generic(SparseGenericArgs a) {
  __shared__ float s_x[kW + kBand];
  const int tid = threadIdx.x;
  const int row = blockIdx.y;
  const long long T0 = (long long)blockIdx.x * kW;
  const float* x = a.x + (long long)(row / a.rows_per_x) * a.x_pitch;
  const int2* tp = a.taps + (long long)row * a.tap_stride;
  const int nnz = a.row_nnz[row];
  float acc[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[r] = 0.f;
  int k = 0;
  while (k < nnz) {
    const int b0 = tp[k].x;  // band covers offsets [b0, b0 + kBand)
    __syncthreads();
    // s_x[i] = x[T0 - b0 - kBand + 1 + i]
    const long long xs = T0 - b0 - kBand + 1;
    for (int i = tid; i < kW + kBand; i += kThreads) {
      const long long t = xs + i;
      s_x[i] = (t >= 0 && t < a.nx) ? __ldg(x + t) : 0.f;
    }
    __syncthreads();
    int kk = k;
    for (; kk < nnz; ++kk) {
      const int2 tv = tp[kk];
      const int rel = tv.x - b0;
      if (rel >= kBand) break;
      const float v = __int_as_float(tv.y);
      // output t = T0 + tid + 128 r ; x index t - o -> s_x[(kBand - 1 - rel) + tid + 128 r]
#pragma unroll
      for (int r = 0; r < 16; ++r) acc[r] = fmaf(v, s_x[kBand - 1 - rel + tid + 128 * r], acc[r]);
    }
    k = kk;
  }
  float* o = a.out + (long long)row * a.out_pitch;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const long long t = T0 + tid + 128 * r;
    if (t < a.out_len) o[t] = acc[r];
  }
}

cudaError_t launch_sparse_generic(const SparseGenericArgs& a, cudaStream_t st) {
  if (a.out_len <= 0 || a.rows <= 0) return cudaSuccess;
  const long long tiles = (a.out_len + kW - 1) / kW;
  k_sparse_generic<<<dim3((unsigned)tiles, (unsigned)a.rows), kThreads, 0, st>>>(a);
  return cudaGetLastError();
}

// ----------------------------------------------------------- g-first mix ----
// Work item = (source group, time tile).  Sources are visited in direction-
// sorted order (a.steps), and the time tiles of all sources that share a
// direction are summed before any reflection tap is applied:
//     sum_s y_s * g_{dir(s)} = sum_d g_d * (sum_{s: dir(s)=d} y_s)      (linearity)
// so the TMEM window write and the 2 x nnz taps run once per *direction*
// present in the group, not once per source.
//
// Every warp is its own pipeline: lane 0 streams the warp's 624-sample slice
// of each source tile (cp.async.bulk + mbarrier complete_tx) and, on a
// direction's last source, its two reflection rows into a warp-private
// kMixStages-deep ring, kMixStages-1 sources ahead; the warp adds slices into
// a private accumulator and, per direction, writes its lanes' windows into its
// TMEM lane quarter and runs both ears as one interleaved pair of
// TMEM-load/FFMA chains.  No CTA-wide barrier in the steady state.  Per-ear
// accumulators persist across the group and leave once per item (bulk store).
constexpr int kMixStages = 3;
constexpr int kMixSlice = 32 * kR + 112;  // floats of a tile one warp reads (KWIN <= 112)

struct MixLayout {
  int slice, stage_floats, taps_off, meta_off, warp_floats, accum_off, bars_off, total;
};

__host__ __device__ inline MixLayout mix_layout(int KWIN, int tap_stride) {
  MixLayout L{};
  L.slice = 32 * kR + KWIN;                              // lane windows 16l + [0, 16 + KWIN)
  L.taps_off = (L.slice + 3) & ~3;                        // [2 ears][tap_stride] int2
  L.meta_off = L.taps_off + 4 * tap_stride;               // int4 {first, last, dir, src}
  L.stage_floats = (L.meta_off + 4 + 31) & ~31;
  L.accum_off = kMixStages * L.stage_floats;              // slice sums, then the item's store staging
  const int acc_floats = padded_len(L.slice);             // bank-padded slice sum
  L.warp_floats = L.accum_off + ((acc_floats > 2 * 32 * kR ? acc_floats : 2 * 32 * kR) + 31 & ~31);
  L.bars_off = kWarps * L.warp_floats;                    // [warps][kMixStages] uint64
  L.total = (L.bars_off + 2 * kWarps * kMixStages) * 4 + 128;
  return L;
}

template <int KWIN, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_mix(MixArgs a) {
  constexpr int XH = KWIN + kR;
  constexpr int COLS = kR + KWIN;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  const MixLayout L = mix_layout(KWIN, a.tap_stride);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* wbase = smem + warp * L.warp_floats;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars_off) + warp * kMixStages;
  float* acc_tile = wbase + L.accum_off;  // aliases the output staging `st`
  float* st = acc_tile;

  if (warp == 0) tmem_alloc<COLS>(&s_tbase);
  if (lane == 0) {
    for (int i = 0; i < kMixStages; ++i) mbar_init(&full[i], 1);
    mbar_fence_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);

  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);
  if (it0 >= it1) {
    tmem_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<COLS>(s_tbase);
    return;
  }
  constexpr int SLICE = 32 * kR + KWIN;          // == L.slice
  const int slice_sig0 = 32 * kR * warp - KWIN;  // signal offset of the slice relative to T0

  // ---- producer cursor: (group, tile, position) advanced incrementally; the
  //      group's step entries are read 32 at a time (one coalesced load per
  //      warp, prefetched a chunk ahead) and broadcast by shuffle.
  int p_grp = (int)(it0 / a.n_tiles), p_j = (int)(it0 - (long long)p_grp * a.n_tiles);
  int p_ns = min(a.src_per_group, a.S - p_grp * a.src_per_group);
  int p_s = 0, issued = 0;
  auto load_chunk = [&](int grp, int ns, int base) -> int4 {
    const int i = base + lane;
    return i < ns ? __ldg(a.steps + (long long)grp * a.src_per_group + i) : make_int4(0, 0, 0, 0);
  };
  int4 ent_chunk = load_chunk(p_grp, p_ns, 0);
  auto issue_one = [&]() {
    // all 32 lanes call this (convergent), lane 0 issues
    if (p_s > 0 && (p_s & 31) == 0) ent_chunk = load_chunk(p_grp, p_ns, p_s);
    const int src = __shfl_sync(0xffffffffu, ent_chunk.x, p_s & 31);
    const int dir = __shfl_sync(0xffffffffu, ent_chunk.y, p_s & 31);
    const int flags = __shfl_sync(0xffffffffu, ent_chunk.z | (ent_chunk.w << 1), p_s & 31);
    if (lane == 0) {
      const int stage = issued % kMixStages;
      float* tile = wbase + stage * L.stage_floats;
      const int last = flags >> 1;
      const long long w0 = (long long)p_j * kW + slice_sig0;  // signal index of slice[0]
      const float* y = a.y + (long long)src * a.y_pitch;
      int nb;
      if (w0 >= 0 && w0 + SLICE <= a.T) {
        nb = SLICE & ~3;
        for (int i = nb; i < SLICE; ++i) tile[i] = __ldg(y + w0 + i);
      } else {  // signal edges: zero padding
        const long long lo = max(w0, 0LL), hi = min(w0 + SLICE, a.T);
        const int n = (int)max(hi - lo, 0LL);
        nb = n & ~3;
        for (int i = 0; i < SLICE; ++i) {
          const long long t = w0 + i;
          if (t < lo || t >= lo + nb) tile[i] = (t >= 0 && t < a.T) ? __ldg(y + t) : 0.f;
        }
      }
      const long long lo = max(w0, 0LL);
      *reinterpret_cast<int4*>(tile + L.meta_off) = make_int4(flags & 1, last, dir, src);
      const unsigned tap_bytes = last ? 2u * a.tap_stride * 8u : 0u;
      mbar_arrive_expect_tx(&full[stage], (unsigned)nb * 4u + tap_bytes);
      if (nb) bulk_load(tile + (lo - w0), y + lo, (unsigned)nb * 4u, &full[stage]);
      if (last) {
        int2* taps = reinterpret_cast<int2*>(tile + L.taps_off);
        for (int e = 0; e < 2; ++e) {
          const int ee = e < a.ears ? e : 0;
          bulk_load(taps + e * a.tap_stride, a.taps + ((long long)ee * a.dirs + dir) * a.tap_stride,
                    (unsigned)a.tap_stride * 8u, &full[stage]);
        }
      }
    }
    ++issued;
    if (++p_s == p_ns) {
      p_s = 0;
      if (++p_j == a.n_tiles) {
        p_j = 0;
        ++p_grp;
        p_ns = p_grp < a.groups ? min(a.src_per_group, a.S - p_grp * a.src_per_group) : 0;
      }
      if (p_ns > 0) ent_chunk = load_chunk(p_grp, p_ns, 0);
    }
  };
  long long total = 0;
  {
    int g = (int)(it0 / a.n_tiles), j = (int)(it0 - (long long)g * a.n_tiles);
    for (long long it = it0; it < it1; ++it) {
      total += min(a.src_per_group, a.S - g * a.src_per_group);
      if (++j == a.n_tiles) {
        j = 0;
        ++g;
      }
    }
  }
  while (issued < min((long long)kMixStages - 1, total)) issue_one();

  int step = 0, stage = 0;
  unsigned phase = 0;
  int c_grp = (int)(it0 / a.n_tiles), c_j = (int)(it0 - (long long)c_grp * a.n_tiles);
  for (long long item = it0; item < it1; ++item) {
    const int j = c_j, grp = c_grp;
    if (++c_j == a.n_tiles) {
      c_j = 0;
      ++c_grp;
    }
    const long long T0 = (long long)j * kW;
    const int ns = min(a.src_per_group, a.S - grp * a.src_per_group);
    float accA[16], accB[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      accA[r] = 0.f;
      accB[r] = 0.f;
    }
    for (int s = 0; s < ns; ++s, ++step) {
      if (issued < total) issue_one();  // refills the stage this warp released last step
      mbar_wait(&full[stage], phase);
      const float* tile = wbase + stage * L.stage_floats;
      if (++stage == kMixStages) {
        stage = 0;
        phase ^= 1u;
      }
      const int4 meta = *reinterpret_cast<const int4*>(tile + L.meta_off);
      if (s == 0) {  // the previous item's bulk store may still be reading acc_tile
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      // sum this direction's sources over the warp's slice into a bank-padded
      // accumulator (coalesced, conflict-free), so that the per-lane window
      // reads below (lane stride 16 floats) are conflict-free too
      if (meta.x) {
#pragma unroll
        for (int i = 4 * lane; i < SLICE; i += 128)
          *reinterpret_cast<float4*>(&acc_tile[padi(i)]) = *reinterpret_cast<const float4*>(&tile[i]);
      } else {
#pragma unroll
        for (int i = 4 * lane; i < SLICE; i += 128) {
          float4 acc4 = *reinterpret_cast<const float4*>(&acc_tile[padi(i)]);
          const float4 t4 = *reinterpret_cast<const float4*>(&tile[i]);
          acc4.x += t4.x;
          acc4.y += t4.y;
          acc4.z += t4.z;
          acc4.w += t4.w;
          *reinterpret_cast<float4*>(&acc_tile[padi(i)]) = acc4;
        }
      }
      __syncwarp();
      if (!meta.y) continue;
      // lane windows -> TMEM (previous direction's loads were all waited)
      {
#pragma unroll
        for (int c = 0; c < COLS; c += 16) {
          float v[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t4 = *reinterpret_cast<const float4*>(&acc_tile[padi(16 * lane + c + 4 * q)]);
            v[4 * q] = t4.x;
            v[4 * q + 1] = t4.y;
            v[4 * q + 2] = t4.z;
            v[4 * q + 3] = t4.w;
          }
          tmem_st16(tlane + c, v);
        }
        tmem_wait_st();
      }
      const int2* tA = reinterpret_cast<const int2*>(tile + L.taps_off);
      const int2* tB = tA + a.tap_stride;
      const float keepB = a.ears > 1 ? 1.f : 0.f;
      if constexpr (NNZT > 0) {
        float XA0[16], XB0[16], XA1[16], XB1[16];
        int2 ta = tA[0], tb = tB[0];
        int2 tan = tA[NNZT > 1 ? 1 : 0], tbn = tB[NNZT > 1 ? 1 : 0];
        tmem_ld16(XA0, tlane + ta.x);
        tmem_ld16(XB0, tlane + tb.x);
#pragma unroll
        for (int k = 0; k < NNZT; ++k) {
          const int2 tann = tA[k + 2 < NNZT ? k + 2 : NNZT - 1];
          const int2 tbnn = tB[k + 2 < NNZT ? k + 2 : NNZT - 1];
          float(&XA)[16] = (k & 1) ? XA1 : XA0;
          float(&XB)[16] = (k & 1) ? XB1 : XB0;
          float(&YA)[16] = (k & 1) ? XA0 : XA1;
          float(&YB)[16] = (k & 1) ? XB0 : XB1;
          const unsigned na = tlane + tan.x, nb = tlane + tbn.x;
          tmem_wait_ld();
          if (k + 1 < NNZT) {
            tmem_ld16(YA, na);
            tmem_ld16(YB, nb);
          }
          const float va = __int_as_float(ta.y), vb = __int_as_float(tb.y) * keepB;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
          ta = tan;
          tb = tbn;
          tan = tann;
          tbn = tbnn;
        }
      } else {
        const int dir = meta.z;
        const int nA = a.row_nnz[dir];
        const int nB = a.ears > 1 ? a.row_nnz[a.dirs + dir] : 0;
        const int nk = max(nA, nB);
        for (int k = 0; k < nk; ++k) {
          const int2 ta = tA[k], tb = tB[k];
          float XA[16], XB[16];
          tmem_ld16(XA, tlane + ta.x);
          tmem_ld16(XB, tlane + tb.x);
          tmem_wait_ld();
          const float va = k < nA ? __int_as_float(ta.y) : 0.f;
          const float vb = k < nB ? __int_as_float(tb.y) : 0.f;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
        }
      }
      __syncwarp();
    }
    // ---- the group's partial for this tile -------------------------------
    const long long out_col = T0 + (long long)warp * 32 * kR;
    if (out_col < a.zlen) {
#pragma unroll
      for (int r = 0; r < 16; r += 4) {
        *reinterpret_cast<float4*>(&st[lane * 16 + r]) = make_float4(accA[r], accA[r + 1], accA[r + 2], accA[r + 3]);
        *reinterpret_cast<float4*>(&st[512 + lane * 16 + r]) =
            make_float4(accB[r], accB[r + 1], accB[r + 2], accB[r + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (elect_one()) {
        for (int e = 0; e < a.ears; ++e)
          bulk_store(a.part + ((long long)grp * a.ears + e) * a.part_pitch + out_col, st + 512 * e, 32 * kR * 4);
      }
    }
  }
  if (lane == 0) bulk_wait_all();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(s_tbase);
}

template <int KWIN, int NNZT>
static cudaError_t launch_mix_t(const MixArgs& a, int sm_count, cudaStream_t st) {
  const int bytes = mix_layout(KWIN, a.tap_stride).total;
  auto kern = k_mix<KWIN, NNZT>;  // 4 warps, one TMEM lane quarter each
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return err;
  // TMEM bounds co-residency (512 / COLS CTAs per SM); shared memory and
  // registers are sized to allow exactly that many.
  int per_sm = 512 / (kR + KWIN);
  if (getenv("TOEP_MIX_PERSM")) per_sm = atoi(getenv("TOEP_MIX_PERSM"));
  long long grid = (long long)sm_count * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, bytes, st>>>(a);
  return cudaGetLastError();
}

template <int KWIN>
static cudaError_t mix_nnz(const MixArgs& a, int sm, cudaStream_t st) {
  if (a.uniform_nnz) {
    switch (a.tap_stride_nnz) {
      case 8: return launch_mix_t<KWIN, 8>(a, sm, st);
      case 16: return launch_mix_t<KWIN, 16>(a, sm, st);
      case 24: return launch_mix_t<KWIN, 24>(a, sm, st);
      case 32: return launch_mix_t<KWIN, 32>(a, sm, st);
      default: break;
    }
  }
  return launch_mix_t<KWIN, 0>(a, sm, st);
}

cudaError_t launch_mix(const MixArgs& a, int kwin, int sm_count, cudaStream_t st) {
  switch (kwin) {
    case 112: return mix_nnz<112>(a, sm_count, st);
    case 240: return mix_nnz<240>(a, sm_count, st);
    case 496: return mix_nnz<496>(a, sm_count, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------ bucketed mix ----
// One pass over the sources, no intermediate per-direction sums in HBM.
// Item = (group of buckets, tile of 2048 z samples); persistent CTAs walk a
// contiguous item range.  Per bucket (all sources of one direction):
//   1. every thread sums its 4-sample columns of the bucket's sources over the
//      tile window x[T0-128, T0+2048) straight from HBM into registers (float4
//      loads, two sources in flight), then stores the sum into a bank-padded
//      shared tile;
//   2. each lane writes its 16+KWIN window into its TMEM lane row;
//   3. both ears' taps run as one interleaved pair of TMEM-load/FFMA2 chains,
//      accumulating the item's z tile in registers.
// 4 CTAs per SM (TMEM 128 columns each) overlap one CTA's loads with the
// others' tap loops.  The item's partial leaves by bulk store.
#ifndef TOEP_MIXB_WADDR
#define TOEP_MIXB_WADDR 0
#endif
#ifndef TOEP_MIXB_FADD2
#define TOEP_MIXB_FADD2 1
#endif
template <int KWIN>
struct MixBCfg {
  static constexpr int COLS = kR + KWIN;
  static constexpr int TILE = kW + COLS;            // window samples of a tile (x[T0 - COLS, T0 + kW))
  static constexpr int V4 = (TILE / 4 + kThreads - 1) / kThreads;  // float4 columns per thread
  static constexpr int SLOTS = 3;                   // prefetched source tiles per bucket (cp.async)
  static constexpr int SLOT_STRIDE = 4 * kThreads * V4;
};
constexpr int kMixBMaxBuckets = 512;   // buckets per group (shared-memory tables)
constexpr int kMixBGroupSrcs = 2048;   // source indices of a group kept in shared memory

struct MixBLayout {
  int tile_off, slot_off, taps_off, bptr_off, bdir_off, bsrc_off, total_bytes;
};

__host__ __device__ inline MixBLayout mixb_layout(int KWIN, int tap_stride) {
  MixBLayout L{};
  const int tile = kW + kR + KWIN;
  const int v4 = (tile / 4 + kThreads - 1) / kThreads;
  L.tile_off = 0;
  int off = (padded_len(tile) + 31) & ~31;
  L.slot_off = off;  // [SLOTS][kThreads * V4] float4, thread-private columns
  off += 3 * 4 * kThreads * v4;
  L.taps_off = off;  // [2][tap_stride] int2
  off += (4 * tap_stride + 3) & ~3;
  L.bptr_off = off;
  off += kMixBMaxBuckets + 4;
  L.bdir_off = off;
  off += kMixBMaxBuckets;
  L.bsrc_off = off;
  off += kMixBGroupSrcs;
  L.total_bytes = off * 4;
  return L;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int KWIN, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_mixb(MixBArgs a) {
  using C = MixBCfg<KWIN>;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  const MixBLayout L = mixb_layout(KWIN, a.tap_stride);
  float* s_tile = smem + L.tile_off;  // padded [TILE]
  float4* s_slot = reinterpret_cast<float4*>(smem + L.slot_off);
  int2* s_taps = reinterpret_cast<int2*>(smem + L.taps_off);
  int* s_bptr = reinterpret_cast<int*>(smem + L.bptr_off);
  int* s_bdir = reinterpret_cast<int*>(smem + L.bdir_off);
  int* s_bsrc = reinterpret_cast<int*>(smem + L.bsrc_off);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tmem_alloc<C::COLS>(&s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);

  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);
  int grp = (int)(it0 / a.n_tiles), j = (int)(it0 - (long long)grp * a.n_tiles);
  int tab_grp = -1, gfirst = 0;
  bool src_in_smem = false;
  float chk0 = 0.f, chk1 = 0.f;  // v*0 accumulates NaN iff some summed sample was inf/NaN
  for (long long item = it0; item < it1; ++item) {
    const int b0 = grp * a.buckets_per_group, nb = min(a.buckets - b0, a.buckets_per_group);
    if (grp != tab_grp) {  // the group's bucket tables -> shared memory
      __syncthreads();
      for (int i = tid; i <= nb; i += kThreads) s_bptr[i] = __ldg(a.bptr + b0 + i);
      for (int i = tid; i < nb; i += kThreads) s_bdir[i] = __ldg(a.bdir + b0 + i);
      gfirst = __ldg(a.bptr + b0);
      const int gn = __ldg(a.bptr + b0 + nb) - gfirst;
      src_in_smem = gn <= kMixBGroupSrcs;
      if (src_in_smem)
        for (int i = tid; i < gn; i += kThreads) s_bsrc[i] = __ldg(a.bsrc + gfirst + i);
      __syncthreads();
      tab_grp = grp;
    }
    auto src_at = [&](int i) { return src_in_smem ? s_bsrc[i - gfirst] : __ldg(a.bsrc + i); };
    const long long T0 = (long long)j * kW;
    const long long x0 = T0 - C::COLS;  // signal index of s_tile[0]
    const bool interior = x0 >= 0 && x0 + C::TILE <= a.T;
    // this thread's float4 columns of bucket k's first SLOTS sources -> its slots
    auto prefetch = [&](int k) {
      const int i0 = s_bptr[k], n = min(s_bptr[k + 1] - i0, C::SLOTS);
      for (int u = 0; u < n; ++u) {
        const float4* ys = reinterpret_cast<const float4*>(a.y + (long long)src_at(i0 + u) * a.y_pitch + x0);
#pragma unroll
        for (int q = 0; q < C::V4; ++q) {
          const int c = tid + q * kThreads;
          if (c < C::TILE / 4) cp_async16(&s_slot[u * (kThreads * C::V4) + c], ys + c);
        }
      }
      cp_async_commit();
    };
    float accA[16], accB[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      accA[r] = 0.f;
      accB[r] = 0.f;
    }
    if (interior && nb > 0) prefetch(0);
    for (int k = 0; k < nb; ++k) {
      const int i0 = s_bptr[k], i1 = s_bptr[k + 1];
      const int dir = s_bdir[k];
      // ---- 1. bucket sum over the tile window -> registers ------------------
      float4 v[C::V4];
#pragma unroll
      for (int q = 0; q < C::V4; ++q) v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (interior) {
        cp_async_wait_all();
        const int n = min(i1 - i0, C::SLOTS);
        for (int u = 0; u < n; ++u) {
#pragma unroll
          for (int q = 0; q < C::V4; ++q) {
            const int c = tid + q * kThreads;
            if (c < C::TILE / 4) {
              const float4 l = s_slot[u * (kThreads * C::V4) + c];
#if TOEP_MIXB_FADD2
              fadd2(v[q].x, v[q].y, l.x, l.y);
              fadd2(v[q].z, v[q].w, l.z, l.w);
#else
              v[q].x += l.x;
              v[q].y += l.y;
              v[q].z += l.z;
              v[q].w += l.w;
#endif
            }
          }
        }
        for (int i = i0 + C::SLOTS; i < i1; ++i) {  // large buckets: the rest straight from HBM
          const float4* ys = reinterpret_cast<const float4*>(a.y + (long long)src_at(i) * a.y_pitch + x0);
#pragma unroll
          for (int q = 0; q < C::V4; ++q) {
            const int c = tid + q * kThreads;
            if (c < C::TILE / 4) {
              const float4 l = __ldcs(ys + c);
              v[q].x += l.x;
              v[q].y += l.y;
              v[q].z += l.z;
              v[q].w += l.w;
            }
          }
        }
      } else {  // signal edges: scalar loads with zero padding
        for (int i = i0; i < i1; ++i) {
          const float* ys = a.y + (long long)src_at(i) * a.y_pitch;
#pragma unroll
          for (int q = 0; q < C::V4; ++q) {
            const int c = tid + q * kThreads;
            if (c < C::TILE / 4) {
              const long long t = x0 + 4 * c;
              v[q].x += (t >= 0 && t < a.T) ? ys[t] : 0.f;
              v[q].y += (t + 1 >= 0 && t + 1 < a.T) ? ys[t + 1] : 0.f;
              v[q].z += (t + 2 >= 0 && t + 2 < a.T) ? ys[t + 2] : 0.f;
              v[q].w += (t + 3 >= 0 && t + 3 < a.T) ? ys[t + 3] : 0.f;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < C::V4; ++q) {
        ffma2(chk0, chk1, v[q].x, v[q].y, 0.f);
        ffma2(chk0, chk1, v[q].z, v[q].w, 0.f);
      }
      __syncthreads();  // every warp finished the previous bucket's window write
      {
        float* tb = s_tile + padi(4 * tid);  // padi(4*(tid + 128q)) = padi(4*tid) + 576q
#pragma unroll
        for (int q = 0; q < C::V4; ++q)
          if (tid + q * kThreads < C::TILE / 4) *reinterpret_cast<float4*>(tb + 576 * q) = v[q];
      }
      for (int i = tid; i < 2 * a.tap_stride; i += kThreads) {
        const int e = i >= a.tap_stride, kk = i - e * a.tap_stride;
        const int ee = e < a.ears ? e : 0;
        s_taps[i] = __ldg(a.taps + ((long long)ee * a.dirs + dir) * a.tap_stride + kk);
      }
      __syncthreads();
      if (interior && k + 1 < nb) prefetch(k + 1);  // next bucket's loads overlap this bucket's taps
      // ---- 2. lane windows -> TMEM -----------------------------------------
      {
        // lane window = s_tile[padi(w0 + m)], w0 = 16 + 16*row, m = 0..COLS-1.  With
        // p = w0 & 16: padi(w0 + m) = padi(w0) + m + 4*(m >> 5) + (p && (m & 16) ? 4 : 0),
        // i.e. two base pointers and compile-time offsets (no per-load index math).
        const int w0 = 16 * tid + 16;
        const float* wb0 = s_tile + padi(w0);
        const float* wb1 = wb0 + ((w0 & 16) ? 4 : 0);
#pragma unroll
        for (int c = 0; c < C::COLS; c += 16) {
          float w[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int m = c + 4 * q;
#if TOEP_MIXB_WADDR
            const float4 t4 = *reinterpret_cast<const float4*>(((m & 16) ? wb1 : wb0) + m + 4 * (m >> 5));
#else
            const float4 t4 = *reinterpret_cast<const float4*>(&s_tile[padi(w0 + m)]);
#endif
            w[4 * q] = t4.x;
            w[4 * q + 1] = t4.y;
            w[4 * q + 2] = t4.z;
            w[4 * q + 3] = t4.w;
          }
          tmem_st16(tlane + c, w);
        }
        tmem_wait_st();
      }
      // ---- 3. both ears' taps ----------------------------------------------
      const int2* tA = s_taps;
      const int2* tB = s_taps + a.tap_stride;
      const float keepB = a.ears > 1 ? 1.f : 0.f;
      if constexpr (NNZT > 0) {
        float XA0[16], XB0[16], XA1[16], XB1[16];
        int2 ta = tA[0], tb = tB[0];
        int2 tan = tA[NNZT > 1 ? 1 : 0], tbn = tB[NNZT > 1 ? 1 : 0];
        tmem_ld16(XA0, tlane + ta.x);
        tmem_ld16(XB0, tlane + tb.x);
#pragma unroll
        for (int k = 0; k < NNZT; ++k) {
          const int2 tann = tA[k + 2 < NNZT ? k + 2 : NNZT - 1];
          const int2 tbnn = tB[k + 2 < NNZT ? k + 2 : NNZT - 1];
          float(&XA)[16] = (k & 1) ? XA1 : XA0;
          float(&XB)[16] = (k & 1) ? XB1 : XB0;
          float(&YA)[16] = (k & 1) ? XA0 : XA1;
          float(&YB)[16] = (k & 1) ? XB0 : XB1;
          const unsigned na = tlane + tan.x, nb = tlane + tbn.x;
          tmem_wait_ld();
          if (k + 1 < NNZT) {
            tmem_ld16(YA, na);
            tmem_ld16(YB, nb);
          }
          const float va = __int_as_float(ta.y), vb = __int_as_float(tb.y) * keepB;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
          ta = tan;
          tb = tbn;
          tan = tann;
          tbn = tbnn;
        }
      } else {
        const int nA = __ldg(a.row_nnz + dir);
        const int nB = a.ears > 1 ? __ldg(a.row_nnz + a.dirs + dir) : 0;
        const int nk = max(nA, nB);
        for (int k = 0; k < nk; ++k) {
          const int2 ta = tA[k], tb = tB[k];
          float XA[16], XB[16];
          tmem_ld16(XA, tlane + ta.x);
          tmem_ld16(XB, tlane + tb.x);
          tmem_wait_ld();
          const float va = k < nA ? __int_as_float(ta.y) : 0.f;
          const float vb = k < nB ? __int_as_float(tb.y) : 0.f;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
        }
      }
    }
    // ---- the group's partial for this tile (once per item: plain stores) ----
    const long long out_col = T0 + (long long)warp * 32 * kR + 16 * lane;
    if (out_col < a.zlen) {
      float4* pA = reinterpret_cast<float4*>(a.part + (long long)grp * a.ears * a.part_pitch + out_col);
#pragma unroll
      for (int r = 0; r < 16; r += 4) pA[r / 4] = make_float4(accA[r], accA[r + 1], accA[r + 2], accA[r + 3]);
      if (a.ears > 1) {
        float4* pB = reinterpret_cast<float4*>(a.part + ((long long)grp * a.ears + 1) * a.part_pitch + out_col);
#pragma unroll
        for (int r = 0; r < 16; r += 4) pB[r / 4] = make_float4(accB[r], accB[r + 1], accB[r + 2], accB[r + 3]);
      }
    }
    if (++j == a.n_tiles) {
      j = 0;
      ++grp;
    }
  }
  const bool bad = !isfinite(chk0 + chk1);
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::COLS>(s_tbase);
}

// ------------------------------------------------- warp-private variant ----
// Same items and buckets as k_mixb, but every warp runs its own pipeline on
// its 512-output quarter: it sums its (512 + KWIN)-sample slice of each source
// (22% halo re-read, HBM is not the binding limit here), writes its lanes'
// windows from a warp-private padded slice, and prefetches the next bucket's
// sources *and* tap rows with cp.async.  No CTA barrier inside the bucket
// loop (only when the group's tables change), so warps drift freely.
constexpr int kMixWGroupSrcs = 1024;

struct MixWLayout {
  int warp_floats, slice_off, slot_off, taps_off, bptr_off, bdir_off, bsrc_off, total_bytes;
};

__host__ __device__ inline MixWLayout mixw_layout(int KWIN, int tap_stride) {
  MixWLayout L{};
  const int slice = 32 * kR + KWIN;
  const int v4 = (slice / 4 + 31) / 32;
  L.slice_off = 0;  // padded [slice]
  int off = (padded_len(slice) + 31) & ~31;
  L.slot_off = off;  // [SLOTS][32 lanes * v4] float4 (lane-private)
  off += 3 * 4 * 32 * v4;
  L.taps_off = off;  // [2 buffers][2 ears][tap_stride] int2
  off += 2 * 2 * 2 * tap_stride;
  L.warp_floats = (off + 31) & ~31;
  off = kWarps * L.warp_floats;
  L.bptr_off = off;
  off += kMixBMaxBuckets + 4;
  L.bdir_off = off;
  off += kMixBMaxBuckets;
  L.bsrc_off = off;
  off += kMixWGroupSrcs;
  L.total_bytes = off * 4;
  return L;
}

template <int KWIN, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_mixw(MixBArgs a) {
  constexpr int COLS = kR + KWIN;
  constexpr int SLICE = 32 * kR + KWIN;
  constexpr int V4 = (SLICE / 4 + 31) / 32;
  constexpr int SLOTS = 3;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  const MixWLayout L = mixw_layout(KWIN, a.tap_stride);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* wb = smem + warp * L.warp_floats;
  float* s_slice = wb + L.slice_off;
  float4* s_slot = reinterpret_cast<float4*>(wb + L.slot_off);
  int2* s_taps = reinterpret_cast<int2*>(wb + L.taps_off);
  int* s_bptr = reinterpret_cast<int*>(smem + L.bptr_off);
  int* s_bdir = reinterpret_cast<int*>(smem + L.bdir_off);
  int* s_bsrc = reinterpret_cast<int*>(smem + L.bsrc_off);
  if (warp == 0) tmem_alloc<COLS>(&s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);

  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);
  int grp = (int)(it0 / a.n_tiles), j = (int)(it0 - (long long)grp * a.n_tiles);
  int tab_grp = -1, gfirst = 0;
  bool src_in_smem = false;
  float chk0 = 0.f, chk1 = 0.f;
  for (long long item = it0; item < it1; ++item) {
    const int b0 = grp * a.buckets_per_group, nb = min(a.buckets - b0, a.buckets_per_group);
    if (grp != tab_grp) {  // the group's bucket tables -> shared memory (all warps at this item)
      __syncthreads();
      for (int i = tid; i <= nb; i += kThreads) s_bptr[i] = __ldg(a.bptr + b0 + i);
      for (int i = tid; i < nb; i += kThreads) s_bdir[i] = __ldg(a.bdir + b0 + i);
      gfirst = __ldg(a.bptr + b0);
      const int gn = __ldg(a.bptr + b0 + nb) - gfirst;
      src_in_smem = gn <= kMixWGroupSrcs;
      if (src_in_smem)
        for (int i = tid; i < gn; i += kThreads) s_bsrc[i] = __ldg(a.bsrc + gfirst + i);
      __syncthreads();
      tab_grp = grp;
    }
    auto src_at = [&](int i) { return src_in_smem ? s_bsrc[i - gfirst] : __ldg(a.bsrc + i); };
    const long long T0 = (long long)j * kW;
    const long long w0 = T0 + (long long)warp * 32 * kR - KWIN;  // signal index of s_slice[0]
    const bool interior = w0 >= 0 && w0 + SLICE <= a.T;
    auto prefetch = [&](int k) {  // bucket k's first SLOTS sources (lane columns) and its two tap rows
      const int i0 = s_bptr[k], n = min(s_bptr[k + 1] - i0, SLOTS);
      if (interior) {
        for (int u = 0; u < n; ++u) {
          const float4* ys = reinterpret_cast<const float4*>(a.y + (long long)src_at(i0 + u) * a.y_pitch + w0);
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const int c = lane + 32 * q;
            if (c < SLICE / 4) cp_async16(&s_slot[u * 32 * V4 + c], ys + c);
          }
        }
      }
      const int dir = s_bdir[k];
      int2* tb = s_taps + (k & 1) * 2 * a.tap_stride;
      for (int i = lane; i < a.tap_stride; i += 32) {  // 2 taps (16 B) per copy
        const int e = i >= a.tap_stride / 2, kk = 2 * (i - e * (a.tap_stride / 2));
        const int ee = e < a.ears ? e : 0;
        cp_async16(tb + e * a.tap_stride + kk, a.taps + ((long long)ee * a.dirs + dir) * a.tap_stride + kk);
      }
      cp_async_commit();
    };
    float accA[16], accB[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      accA[r] = 0.f;
      accB[r] = 0.f;
    }
    if (nb > 0) prefetch(0);
    for (int k = 0; k < nb; ++k) {
      const int i0 = s_bptr[k], i1 = s_bptr[k + 1];
      float4 v[V4];
#pragma unroll
      for (int q = 0; q < V4; ++q) v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      cp_async_wait_all();
      if (interior) {
        const int n = min(i1 - i0, SLOTS);
        for (int u = 0; u < n; ++u) {
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const int c = lane + 32 * q;
            if (c < SLICE / 4) {
              const float4 l = s_slot[u * 32 * V4 + c];
              fadd2(v[q].x, v[q].y, l.x, l.y);
              fadd2(v[q].z, v[q].w, l.z, l.w);
            }
          }
        }
        for (int i = i0 + SLOTS; i < i1; ++i) {
          const float4* ys = reinterpret_cast<const float4*>(a.y + (long long)src_at(i) * a.y_pitch + w0);
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const int c = lane + 32 * q;
            if (c < SLICE / 4) {
              const float4 l = __ldcs(ys + c);
              fadd2(v[q].x, v[q].y, l.x, l.y);
              fadd2(v[q].z, v[q].w, l.z, l.w);
            }
          }
        }
      } else {
        for (int i = i0; i < i1; ++i) {
          const float* ys = a.y + (long long)src_at(i) * a.y_pitch;
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const int c = lane + 32 * q;
            if (c < SLICE / 4) {
              const long long t = w0 + 4 * c;
              v[q].x += (t >= 0 && t < a.T) ? ys[t] : 0.f;
              v[q].y += (t + 1 >= 0 && t + 1 < a.T) ? ys[t + 1] : 0.f;
              v[q].z += (t + 2 >= 0 && t + 2 < a.T) ? ys[t + 2] : 0.f;
              v[q].w += (t + 3 >= 0 && t + 3 < a.T) ? ys[t + 3] : 0.f;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < V4; ++q) {
        ffma2(chk0, chk1, v[q].x, v[q].y, 0.f);
        ffma2(chk0, chk1, v[q].z, v[q].w, 0.f);
      }
      __syncwarp();  // previous bucket's window reads of s_slice are done; tap rows of k visible
      {
        float* sb = s_slice + padi(4 * lane);  // padi(4*(lane + 32q)) = padi(4*lane) + 144q
#pragma unroll
        for (int q = 0; q < V4; ++q)
          if (lane + 32 * q < SLICE / 4) *reinterpret_cast<float4*>(sb + 144 * q) = v[q];
      }
      __syncwarp();
      const int2* tA = s_taps + (k & 1) * 2 * a.tap_stride;
      const int2* tB = tA + a.tap_stride;
      const int dir = s_bdir[k];
      if (k + 1 < nb) prefetch(k + 1);  // next bucket's loads overlap this bucket's taps
      {
#pragma unroll
        for (int c = 0; c < COLS; c += 16) {
          float w[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t4 = *reinterpret_cast<const float4*>(&s_slice[padi(16 * lane + c + 4 * q)]);
            w[4 * q] = t4.x;
            w[4 * q + 1] = t4.y;
            w[4 * q + 2] = t4.z;
            w[4 * q + 3] = t4.w;
          }
          tmem_st16(tlane + c, w);
        }
        tmem_wait_st();
      }
      const float keepB = a.ears > 1 ? 1.f : 0.f;
      if constexpr (NNZT > 0) {
        float XA0[16], XB0[16], XA1[16], XB1[16];
        int2 ta = tA[0], tb = tB[0];
        int2 tan = tA[NNZT > 1 ? 1 : 0], tbn = tB[NNZT > 1 ? 1 : 0];
        tmem_ld16(XA0, tlane + ta.x);
        tmem_ld16(XB0, tlane + tb.x);
#pragma unroll
        for (int kk = 0; kk < NNZT; ++kk) {
          const int2 tann = tA[kk + 2 < NNZT ? kk + 2 : NNZT - 1];
          const int2 tbnn = tB[kk + 2 < NNZT ? kk + 2 : NNZT - 1];
          float(&XA)[16] = (kk & 1) ? XA1 : XA0;
          float(&XB)[16] = (kk & 1) ? XB1 : XB0;
          float(&YA)[16] = (kk & 1) ? XA0 : XA1;
          float(&YB)[16] = (kk & 1) ? XB0 : XB1;
          const unsigned na = tlane + tan.x, nb2 = tlane + tbn.x;
          tmem_wait_ld();
          if (kk + 1 < NNZT) {
            tmem_ld16(YA, na);
            tmem_ld16(YB, nb2);
          }
          const float va = __int_as_float(ta.y), vb = __int_as_float(tb.y) * keepB;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
          ta = tan;
          tb = tbn;
          tan = tann;
          tbn = tbnn;
        }
      } else {
        const int nA = __ldg(a.row_nnz + dir);
        const int nB = a.ears > 1 ? __ldg(a.row_nnz + a.dirs + dir) : 0;
        const int nk = max(nA, nB);
        for (int kk = 0; kk < nk; ++kk) {
          const int2 ta = tA[kk], tb = tB[kk];
          float XA[16], XB[16];
          tmem_ld16(XA, tlane + ta.x);
          tmem_ld16(XB, tlane + tb.x);
          tmem_wait_ld();
          const float va = kk < nA ? __int_as_float(ta.y) : 0.f;
          const float vb = kk < nB ? __int_as_float(tb.y) : 0.f;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
        }
      }
    }
    const long long out_col = T0 + (long long)warp * 32 * kR + 16 * lane;
    if (out_col < a.zlen) {
      float4* pA = reinterpret_cast<float4*>(a.part + (long long)grp * a.ears * a.part_pitch + out_col);
#pragma unroll
      for (int r = 0; r < 16; r += 4) pA[r / 4] = make_float4(accA[r], accA[r + 1], accA[r + 2], accA[r + 3]);
      if (a.ears > 1) {
        float4* pB = reinterpret_cast<float4*>(a.part + ((long long)grp * a.ears + 1) * a.part_pitch + out_col);
#pragma unroll
        for (int r = 0; r < 16; r += 4) pB[r / 4] = make_float4(accB[r], accB[r + 1], accB[r + 2], accB[r + 3]);
      }
    }
    if (++j == a.n_tiles) {
      j = 0;
      ++grp;
    }
  }
  cp_async_wait_all();
  const bool bad = !isfinite(chk0 + chk1);
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(s_tbase);
}

template <int KWIN, int NNZT>
static cudaError_t launch_mixb_t(const MixBArgs& a, int sm_count, cudaStream_t st) {
  static const bool warp_private = [] {
    const char* ev = getenv("TOEP_MIX_KERNEL");
    return !(ev && ev[0] == 'b');
  }();
  const int bytes = warp_private ? mixw_layout(KWIN, a.tap_stride).total_bytes
                                 : mixb_layout(KWIN, a.tap_stride).total_bytes;
  auto kern = warp_private ? k_mixw<KWIN, NNZT> : k_mixb<KWIN, NNZT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return err;
  long long grid = (long long)sm_count * (512 / (kR + KWIN));  // TMEM-bounded co-residency
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, bytes, st>>>(a);
  return cudaGetLastError();
}

template <int KWIN>
static cudaError_t mixb_nnz(const MixBArgs& a, int nnz_uniform, int sm, cudaStream_t st) {
  switch (nnz_uniform) {
    case 8: return launch_mixb_t<KWIN, 8>(a, sm, st);
    case 16: return launch_mixb_t<KWIN, 16>(a, sm, st);
    case 24: return launch_mixb_t<KWIN, 24>(a, sm, st);
    case 32: return launch_mixb_t<KWIN, 32>(a, sm, st);
    default: return launch_mixb_t<KWIN, 0>(a, sm, st);
  }
}

cudaError_t launch_mixb(const MixBArgs& a, int kwin, int nnz_uniform, int sm_count, cudaStream_t st) {
  switch (kwin) {
    case 112: return mixb_nnz<112>(a, nnz_uniform, sm_count, st);
    case 240: return mixb_nnz<240>(a, nnz_uniform, sm_count, st);
    case 496: return mixb_nnz<496>(a, nnz_uniform, sm_count, st);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------ same-direction source sums ----
// yb[b][t] = sum over the sources of bucket b (all at one direction) of y_s[t].
// Pure streaming pass (HBM-bound): float4 loads, up to 4 sources in flight.
__global__ void __launch_bounds__(256) k_bucket_sum(const float* __restrict__ y, long long y_pitch, long long T,
                                                    const int* __restrict__ bsrc, const int* __restrict__ bptr,
                                                    float* __restrict__ yb, long long yb_pitch) {
  const int b = blockIdx.y;
  const int i0 = bptr[b], i1 = bptr[b + 1];
  float* out = yb + (long long)b * yb_pitch;
  const long long n4 = T >> 2;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int i = i0;
    for (; i + 4 <= i1; i += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(y + (long long)bsrc[i + u] * y_pitch) + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x;
        acc.y += v[u].y;
        acc.z += v[u].z;
        acc.w += v[u].w;
      }
    }
    for (; i < i1; ++i) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(y + (long long)bsrc[i] * y_pitch) + q);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[q] = acc;
  }
  if (blockIdx.x == 0) {
    for (long long t = 4 * n4 + threadIdx.x; t < T; t += blockDim.x) {
      float acc = 0.f;
      for (int i = i0; i < i1; ++i) acc += y[(long long)bsrc[i] * y_pitch + t];
      out[t] = acc;
    }
  }
}

cudaError_t launch_bucket_sum(const float* y, long long y_pitch, long long T, const int* bsrc, const int* bptr,
                              int buckets, float* yb, long long yb_pitch, int sm_count, cudaStream_t st) {
  const long long n4 = T >> 2;
  long long bx = (n4 + 255) / 256;
  const long long cap = std::max(1LL, (long long)sm_count * 8 / std::max(1, buckets) + 1);
  if (bx > cap * 64) bx = cap * 64;
  if (bx < 1) bx = 1;
  k_bucket_sum<<<dim3((unsigned)bx, (unsigned)buckets), 256, 0, st>>>(y, y_pitch, T, bsrc, bptr, yb, yb_pitch);
  return cudaGetLastError();
}

__global__ void k_mix_reduce(const float* __restrict__ part, int groups, int ears, long long part_pitch,
                             long long zlen, float* __restrict__ z, long long z_pitch) {
  const int e = blockIdx.y;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < zlen;
       t += (long long)gridDim.x * blockDim.x) {
    // pairwise over groups: sum adjacent pairs first (fixed order)
    float acc = 0.f;
    int g = 0;
    for (; g + 1 < groups; g += 2)
      acc += part[((long long)g * ears + e) * part_pitch + t] + part[((long long)(g + 1) * ears + e) * part_pitch + t];
    if (g < groups) acc += part[((long long)g * ears + e) * part_pitch + t];
    z[(long long)e * z_pitch + t] = acc;
  }
}

cudaError_t launch_mix_reduce(const float* part, int groups, int ears, long long part_pitch, long long zlen,
                              float* z, long long z_pitch, cudaStream_t st) {
  if (zlen <= 0) return cudaSuccess;
  long long blocks = (zlen + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_mix_reduce<<<dim3((unsigned)blocks, (unsigned)ears), 256, 0, st>>>(part, groups, ears, part_pitch, zlen, z,
                                                                       z_pitch);
  return cudaGetLastError();
}

// ------------------------------------------------------ streaming block ----
// One launch per block of B <= 256 samples (latency path).  CTA c owns
// src_per_cta sources; thread t owns output sample t for both ears.  The CTA
// loads its sources' [history | block] windows and tap rows into shared
// memory in one vectorised round, accumulates per-thread (3 instructions per
// tap: broadcast tap, window sample, FFMA), writes one partial and rolls the
// sources' history.  Partials are reduced deterministically in two ticketed
// levels (groups of kStreamGroup CTAs, then the groups), and the very last CTA
// applies f_e over [z history | z block] and rolls the z history.
constexpr int kStreamGroup = 16;

__device__ __forceinline__ bool stream_last_arrival(unsigned int* ticket, unsigned int n) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == n - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

__global__ void __launch_bounds__(256) k_stream_step(StreamArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  const int L = a.H + a.B;  // multiple of 4 (host checks)
  const int s0 = blockIdx.x * a.src_per_cta;
  const int ns = min(a.S - s0, a.src_per_cta);
  float* s_w = sm;                                                // [ns][L]
  int2* s_tap = reinterpret_cast<int2*>(sm + a.src_per_cta * L);  // [ns][ears][tap_stride]
  int* s_nnz = reinterpret_cast<int*>(s_tap + a.src_per_cta * a.ears * a.tap_stride);
  float chk = 0.f;  // fused DataError check on the new block's samples
  {
    const int q4 = L / 4, h4 = a.H / 4;
    for (int i = tid; i < ns * q4; i += blockDim.x) {
      const int s = i / q4, q = i - s * q4;
      float4 v;
      if (q < h4) {
        v = *reinterpret_cast<const float4*>(a.yhist + (long long)(s0 + s) * a.H + 4 * q);
      } else {
        v = __ldg(reinterpret_cast<const float4*>(a.block + (long long)(s0 + s) * a.block_pitch) + (q - h4));
        chk = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, chk))));
      }
      *reinterpret_cast<float4*>(&s_w[s * L + 4 * q]) = v;
    }
    for (int i = tid; i < ns * a.ears * a.tap_stride; i += blockDim.x) {
      const int se = i / a.tap_stride, k = i - se * a.tap_stride;
      const int s = se / a.ears, e = se - s * a.ears;
      const long long row = (long long)e * a.dirs + a.src_dir[s0 + s];
      s_tap[i] = a.taps[row * a.tap_stride + k];
      if (k == 0) s_nnz[se] = a.row_nnz[row];
    }
  }
  __syncthreads();
  const int t = tid;
  float acc0 = 0.f, acc1 = 0.f;
  if (t < a.B) {
    for (int s = 0; s < ns; ++s) {
      const float* w = s_w + s * L + a.H + t;
      const int2* t0 = s_tap + (s * a.ears) * a.tap_stride;
      const int n0 = s_nnz[s * a.ears];
#pragma unroll 4
      for (int k = 0; k < n0; ++k) acc0 = fmaf(__int_as_float(t0[k].y), w[-t0[k].x], acc0);
      if (a.ears > 1) {
        const int2* t1 = t0 + a.tap_stride;
        const int n1 = s_nnz[s * a.ears + 1];
#pragma unroll 4
        for (int k = 0; k < n1; ++k) acc1 = fmaf(__int_as_float(t1[k].y), w[-t1[k].x], acc1);
      }
    }
    a.part[((long long)blockIdx.x * a.ears) * a.B + t] = acc0;
    if (a.ears > 1) a.part[((long long)blockIdx.x * a.ears + 1) * a.B + t] = acc1;
  }
  if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && (tid & 31) == 0) atomicOr(a.nonfinite, 1);
  // roll the sources' history: keep the last H samples of [hist | block]
  for (int i = tid; i < ns * (a.H / 4); i += blockDim.x) {
    const int s = i / (a.H / 4), q = i - s * (a.H / 4);
    *reinterpret_cast<float4*>(a.yhist + (long long)(s0 + s) * a.H + 4 * q) =
        *reinterpret_cast<const float4*>(&s_w[s * L + a.B + 4 * q]);
  }
  // ---- level 1: the last CTA of each group sums the group's partials --------
  const int groups = (gridDim.x + kStreamGroup - 1) / kStreamGroup;
  const int grp = blockIdx.x / kStreamGroup;
  const int c0 = grp * kStreamGroup, nc = min((int)gridDim.x - c0, kStreamGroup);
  if (!stream_last_arrival(a.ticket + grp, nc)) return;
  const long long cs = (long long)a.ears * a.B;
  for (int i = tid; i < a.ears * a.B; i += blockDim.x) {
    float z[kStreamGroup];
#pragma unroll
    for (int u = 0; u < kStreamGroup; ++u) z[u] = u < nc ? __ldcg(a.part + (c0 + u) * cs + i) : 0.f;
#pragma unroll
    for (int w = kStreamGroup / 2; w > 0; w /= 2)
#pragma unroll
      for (int u = 0; u < w; ++u) z[u] += z[u + w];
    a.gpart[grp * cs + i] = z[0];
  }
  if (tid == 0) a.ticket[grp] = 0u;
  // ---- level 2: the last group finishes: z = sum of groups, out = f * z -----
  if (!stream_last_arrival(a.ticket + groups, groups)) return;
  float* s_z = sm;                          // [ears][zh + B]
  float* s_f = sm + a.ears * (a.zh + a.B);  // [ears][lf_pad]
  for (int i = tid; i < a.ears * a.zh; i += blockDim.x) {
    const int e = i / a.zh, k = i - e * a.zh;
    s_z[e * (a.zh + a.B) + k] = a.zhist[(long long)e * a.zh + k];
  }
  for (int i = tid; i < a.ears * a.lf_pad; i += blockDim.x) s_f[i] = a.f[i];
  for (int i = tid; i < a.ears * a.B; i += blockDim.x) {
    const int e = i / a.B, tt = i - e * a.B;
    float z = 0.f;
    for (int g = 0; g < groups; ++g) z += __ldcg(a.gpart + g * cs + i);
    s_z[e * (a.zh + a.B) + a.zh + tt] = z;
  }
  __syncthreads();
  for (int i = tid; i < a.ears * a.B; i += blockDim.x) {
    const int e = i / a.B, tt = i - e * a.B;
    const float* z = s_z + e * (a.zh + a.B) + a.zh + tt;
    const float* ff = s_f + e * a.lf_pad;
    float o = 0.f;
#pragma unroll 8
    for (int jj = 0; jj < a.lf_pad; ++jj) o = fmaf(ff[jj], z[-jj], o);
    a.out[(long long)e * a.out_pitch + tt] = o;
  }
  __syncthreads();
  for (int i = tid; i < a.ears * a.zh; i += blockDim.x) {
    const int e = i / a.zh, k = i - e * a.zh;
    a.zhist[(long long)e * a.zh + k] = s_z[e * (a.zh + a.B) + a.B + k];
  }
  if (tid == 0) a.ticket[groups] = 0u;
}

cudaError_t launch_stream_step(const StreamArgs& a, cudaStream_t st) {
  const size_t per_cta = (size_t)a.src_per_cta * (a.H + a.B) + (size_t)a.src_per_cta * a.ears * a.tap_stride * 2 +
                         (size_t)a.src_per_cta * a.ears;
  const size_t fin = (size_t)a.ears * (a.zh + a.B + a.lf_pad);
  const size_t smem = std::max(per_cta, fin) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_stream_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_stream_step<<<a.ctas, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace toep
