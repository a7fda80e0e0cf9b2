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
// sorted order (a.order), and the time tiles of all sources that share a
// direction are summed before any reflection tap is applied:
//     sum_s y_s * g_{dir(s)} = sum_d g_d * (sum_{s: dir(s)=d} y_s)      (linearity)
// so the TMEM window write and the 2 x nnz taps run once per *direction*
// present in the group, not once per source.
//
// Pipeline: a producer warp streams each source's window tile (cp.async.bulk
// with mbarrier completion) plus the two reflection rows of its direction into
// a kMixStages-deep shared-memory ring.  The 4 consumer warps each add their
// 624-sample slice of the tile into a warp-private accumulator, release the
// stage, and on the last source of a direction write their lanes' windows into
// their TMEM lane quarter and run both ears as one interleaved pair of
// TMEM-load/FFMA chains.  Per-ear accumulators persist across the group and
// leave once per item through a bulk store.
constexpr int kMixStages = 6;
constexpr int kMixThreads = kThreads + 32;  // 4 consumer warps + 1 TMA producer warp
constexpr int kMixSlice = 32 * kR + 128;   // floats of the tile one warp needs (<= 512 + KWIN + 16)

struct MixLayout {
  int stage_floats, taps_off, meta_off, steps_off, staging_off, accum_off, bars_off, total;
};

__host__ __device__ inline MixLayout mix_layout(int KWIN, int tap_stride) {
  MixLayout L{};
  const int XH = KWIN + kR;
  const int tile = (kW + XH + 31) & ~31;
  const int slice = 32 * kR + XH;
  L.taps_off = tile;                      // within a stage: [2 ears][tap_stride] int2
  L.meta_off = tile + 4 * tap_stride;     // int4 {first, last, dir, src}
  L.stage_floats = (L.meta_off + 4 + 31) & ~31;
  L.steps_off = kMixStages * L.stage_floats;             // int4 [src_per_group] producer step table
  L.accum_off = L.steps_off + 4 * 256;                    // [warps][slice]
  L.staging_off = L.accum_off + kWarps * ((slice + 31) & ~31);  // [warps][2 ears][512]
  L.bars_off = L.staging_off + kWarps * 2 * 32 * kR;        // 2*kMixStages uint64
  L.total = (L.bars_off + 4 * kMixStages) * 4 + 128;
  return L;
}

__device__ __forceinline__ int mix_group_size(const MixArgs& a, long long item) {
  const int grp = (int)(item / a.n_tiles);
  return min(a.src_per_group, a.S - grp * a.src_per_group);
}

// Prefetch one (item, source) step into its ring stage (producer lane 0).
// `ent` = {src, dir, first, last} from the host-built direction-sorted table.
template <int KWIN>
__device__ __forceinline__ void mix_issue(const MixArgs& a, const MixLayout& L, float* smem, uint64_t* full,
                                          uint64_t* empty, int j, int4 ent, int issued) {
  constexpr int XH = KWIN + kR;
  const int stage = issued % kMixStages;
  const unsigned par = (unsigned)((issued / kMixStages) & 1);
  mbar_wait(&empty[stage], par ^ 1u);
  const int src = ent.x, dir = ent.y, last = ent.w;
  float* tile = smem + stage * L.stage_floats;
  int2* taps = reinterpret_cast<int2*>(tile + L.taps_off);
  const long long T0 = (long long)j * kW;
  const long long w0 = T0 - XH;  // signal index of tile[0]
  const long long lo = max(w0, 0LL), hi = min(T0 + kW, a.T);
  const int n = (int)max(hi - lo, 0LL);
  const int nb = n & ~3;
  const unsigned tap_bytes = last ? 2u * a.tap_stride * 8u : 0u;
  const float* y = a.y + (long long)src * a.y_pitch;
  // zero fill / ragged remainder / metadata with generic stores, released by the arrive below
  for (long long i = 0; i < lo - w0; ++i) tile[i] = 0.f;
  for (int i = nb; i < n; ++i) tile[(lo - w0) + i] = __ldg(y + lo + i);
  for (long long i = (lo - w0) + n; i < kW + XH; ++i) tile[i] = 0.f;
  *reinterpret_cast<int4*>(tile + L.meta_off) = make_int4(ent.z, ent.w, dir, src);
  mbar_arrive_expect_tx(&full[stage], (unsigned)nb * 4u + tap_bytes);
  if (nb) bulk_load(tile + (lo - w0), y + lo, (unsigned)nb * 4u, &full[stage]);
  if (last) {
    for (int e = 0; e < 2; ++e) {
      const int ee = e < a.ears ? e : 0;
      bulk_load(taps + e * a.tap_stride, a.taps + ((long long)ee * a.dirs + dir) * a.tap_stride,
                (unsigned)a.tap_stride * 8u, &full[stage]);
    }
  }
}

template <int KWIN, int NNZT>
__global__ void __maxnreg__(136) k_mix(MixArgs a) {
  constexpr int XH = KWIN + kR;
  constexpr int COLS = kR + KWIN;
  constexpr int SLICE = 32 * kR + KWIN;  // tile floats one warp reads (lane windows 16l + [0, 128))
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  const MixLayout L = mix_layout(KWIN, a.tap_stride);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars_off);
  uint64_t* empty = full + kMixStages;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tmem_alloc<COLS>(&s_tbase);
  if (tid == 0) {
    for (int i = 0; i < kMixStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kWarps);
    }
    mbar_fence_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * (warp & 3)) << 16);

  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);

  if (warp == kWarps) {
    // ---- producer warp: streams every (item, source) of this CTA into the ring;
    //      the group's step table is staged in shared memory once per group
    int4* s_steps = reinterpret_cast<int4*>(smem + L.steps_off);
    int issued = 0, cur_grp = -1;
    for (long long item = it0; item < it1; ++item) {
      const int j = (int)(item % a.n_tiles);
      const int grp = (int)(item / a.n_tiles);
      const int ns = mix_group_size(a, item);
      if (grp != cur_grp) {
        __syncwarp();
        for (int i = lane; i < ns; i += 32) s_steps[i] = a.steps[(long long)grp * a.src_per_group + i];
        __syncwarp();
        cur_grp = grp;
      }
      if (lane == 0)
        for (int s = 0; s < ns; ++s, ++issued) mix_issue<KWIN>(a, L, smem, full, empty, j, s_steps[s], issued);
      __syncwarp();
    }
  } else {
    int step = 0;
    float* st = smem + L.staging_off + warp * 2 * 32 * kR;
    float* acc_tile = smem + L.accum_off + warp * ((SLICE + 31) & ~31);
    const int slice0 = (XH - KWIN) + 32 * kR * warp;  // this warp's first tile index
    for (long long item = it0; item < it1; ++item) {
      const int j = (int)(item % a.n_tiles);
      const int grp = (int)(item / a.n_tiles);
      const long long T0 = (long long)j * kW;
      const int ns = mix_group_size(a, item);
      float accA[16], accB[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        accA[r] = 0.f;
        accB[r] = 0.f;
      }
      for (int s = 0; s < ns; ++s, ++step) {
        const int stage = step % kMixStages;
        mbar_wait(&full[stage], (unsigned)((step / kMixStages) & 1));
        const float* tile = smem + stage * L.stage_floats;
        const int4 meta = *reinterpret_cast<const int4*>(tile + L.meta_off);
        // sum this direction's sources over the warp's slice (coalesced, conflict-free)
        if (meta.x) {
          for (int i = 4 * lane; i < SLICE; i += 128)
            *reinterpret_cast<float4*>(&acc_tile[i]) = *reinterpret_cast<const float4*>(&tile[slice0 + i]);
        } else {
          for (int i = 4 * lane; i < SLICE; i += 128) {
            float4 acc4 = *reinterpret_cast<const float4*>(&acc_tile[i]);
            const float4 t4 = *reinterpret_cast<const float4*>(&tile[slice0 + i]);
            acc4.x += t4.x;
            acc4.y += t4.y;
            acc4.z += t4.z;
            acc4.w += t4.w;
            *reinterpret_cast<float4*>(&acc_tile[i]) = acc4;
          }
        }
        if (!meta.y) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          continue;
        }
        __syncwarp();
        // lane windows -> TMEM (previous direction's loads were all waited)
        {
          const int wbase = 16 * lane;
#pragma unroll
          for (int c = 0; c < COLS; c += 16) {
            float v[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 t4 = *reinterpret_cast<const float4*>(&acc_tile[wbase + c + 4 * q]);
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
            for (int r = 0; r < 16; ++r) {
              accA[r] = fmaf(va, XA[r], accA[r]);
              accB[r] = fmaf(vb, XB[r], accB[r]);
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
            for (int r = 0; r < 16; ++r) {
              accA[r] = fmaf(va, XA[r], accA[r]);
              accB[r] = fmaf(vb, XB[r], accB[r]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
      }
      // ---- the group's partial for this tile -----------------------------
      const long long out_col = T0 + (long long)warp * 32 * kR;
      if (out_col < a.zlen) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 16; r += 4) {
          *reinterpret_cast<float4*>(&st[lane * 16 + r]) = make_float4(accA[r], accA[r + 1], accA[r + 2], accA[r + 3]);
          *reinterpret_cast<float4*>(&st[512 + lane * 16 + r]) =
              make_float4(accB[r], accB[r + 1], accB[r + 2], accB[r + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int e = 0; e < a.ears; ++e)
            bulk_store(a.part + ((long long)grp * a.ears + e) * a.part_pitch + out_col, st + 512 * e, 32 * kR * 4);
        }
      }
    }
    if (lane == 0) bulk_wait_all();
  }  // consumer warps
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(s_tbase);
}

template <int KWIN, int NNZT>
static cudaError_t launch_mix_t(const MixArgs& a, int sm_count, cudaStream_t st) {
  const int bytes = mix_layout(KWIN, a.tap_stride).total;
  auto kern = k_mix<KWIN, NNZT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return err;
  const int per_sm = std::min(3, 512 / (kR + KWIN));
  long long grid = (long long)sm_count * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kMixThreads, bytes, st>>>(a);
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
// One launch per block of B samples: every CTA owns src_per_cta sources,
// forms [history | block] windows in shared memory, accumulates both ears'
// partial z over its sources, and rolls the source history forward.  The
// last CTA to finish (atomic ticket) sums the partials in fixed CTA order,
// applies f_e over [z history | z block] and rolls the z history.
__global__ void __launch_bounds__(256) k_stream_step(StreamArgs a) {
  unsigned int* ticket = a.ticket;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  float* s_w = sm;  // [L] window of current source
  __shared__ bool s_last;
  const int s0 = blockIdx.x * a.src_per_cta;
  const int s1 = min(a.S, s0 + a.src_per_cta);
  for (int e = 0; e < a.ears; ++e)
    for (int t = tid; t < a.B; t += blockDim.x) a.part[((long long)blockIdx.x * a.ears + e) * a.B + t] = 0.f;
  float acc[2][4];
  for (int s = s0; s < s1; ++s) {
    __syncthreads();
    for (int i = tid; i < a.H; i += blockDim.x) s_w[i] = a.yhist[(long long)s * a.H + i];
    for (int i = tid; i < a.B; i += blockDim.x) s_w[a.H + i] = a.block[(long long)s * a.B + i];
    __syncthreads();
    const int dir = a.src_dir[s];
    for (int e = 0; e < a.ears; ++e) {
      const long long row = (long long)e * a.dirs + dir;
      const int2* tp = a.taps + row * a.tap_stride;
      const int nnz = a.row_nnz[row];
      for (int q = 0; q < 4; ++q) acc[e][q] = 0.f;
      for (int k = 0; k < nnz; ++k) {
        const int2 tv = tp[k];
        const float v = __int_as_float(tv.y);
        for (int q = 0; q < 4; ++q) {
          const int t = tid + 256 * q;
          if (t < a.B) acc[e][q] = fmaf(v, s_w[a.H + t - tv.x], acc[e][q]);
        }
      }
      for (int q = 0; q < 4; ++q) {
        const int t = tid + 256 * q;
        if (t < a.B) a.part[((long long)blockIdx.x * a.ears + e) * a.B + t] += acc[e][q];
      }
    }
    __syncthreads();
    // roll this source's history: keep the last H samples of [hist | block]
    for (int i = tid; i < a.H; i += blockDim.x) a.yhist[(long long)s * a.H + i] = s_w[a.B + i];
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // z window per ear: [zhist (zh) | zblock (B)], out = f * z over the block
  float* s_z = sm;
  float* s_f = sm + (a.zh + a.B);
  for (int e = 0; e < a.ears; ++e) {
    __syncthreads();
    for (int i = tid; i < a.zh; i += blockDim.x) s_z[i] = a.zhist[(long long)e * a.zh + i];
    for (int t = tid; t < a.B; t += blockDim.x) {
      float zz = 0.f;
      for (int c = 0; c < gridDim.x; ++c) zz += a.part[((long long)c * a.ears + e) * a.B + t];
      s_z[a.zh + t] = zz;
    }
    for (int i = tid; i < a.lf_pad; i += blockDim.x) s_f[i] = a.f[(long long)e * a.lf_pad + i];
    __syncthreads();
    for (int t = tid; t < a.B; t += blockDim.x) {
      float o = 0.f;
      for (int jj = 0; jj < a.lf_pad; ++jj) o = fmaf(s_f[jj], s_z[a.zh + t - jj], o);
      a.out[(long long)e * a.B + t] = o;
    }
    __syncthreads();
    for (int i = tid; i < a.zh; i += blockDim.x) a.zhist[(long long)e * a.zh + i] = s_z[a.B + i];
  }
  if (tid == 0) *ticket = 0u;
}

cudaError_t launch_stream_step(const StreamArgs& a, cudaStream_t st) {
  const size_t smem = (size_t)max(a.H + a.B, a.zh + a.B + a.lf_pad) * 4;
  k_stream_step<<<a.ctas, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace toep
