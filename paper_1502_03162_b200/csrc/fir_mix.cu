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
    for (int i = tid; i < nch; i += kThreads) s_h[i] = j0 + i < a.nh ? h[j0 + i] : 0.f;
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

// --------------------------------------------------------- mixdown ----
// One pass over the sources; no intermediate per-direction sums in HBM.
// Buckets are the sets of sources sharing a direction (host stable sort).
// Item = (group of buckets, 2048-sample z tile); persistent CTAs (4 per SM,
// TMEM 128 columns each) walk contiguous item ranges, the group's bucket
// tables sit in shared memory.  Every warp runs its own pipeline on its
// 512-output quarter of the tile, per bucket (all sources of one direction):
//   1. sum its (512 + KWIN)-sample slice of the bucket's sources into
//      registers (the first 3 sources were prefetched with cp.async into
//      lane-private shared-memory slots while the previous bucket's taps ran;
//      the rest stream straight from HBM), store the sum into a warp-private
//      bank-padded slice;
//   2. each lane writes its 16+KWIN window into its TMEM lane row;
//   3. both ears' taps (ear-interleaved int4 table, prefetched with the
//      sources) run as one interleaved pair of TMEM-load/FFMA2 chains,
//      accumulating the item's z quarter in registers.
// No CTA barrier inside the bucket loop (only when the group's tables
// change), so warps drift freely; partials leave once per item.


__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }


constexpr int kMixSlots = 4;
  // sources per bucket prefetched into shared-memory slots

struct MixLayout {
  int warp_floats, slot_floats, slot_off, taps_off, bptr_off, bdir_off, boff_off, total_bytes;
};

// Per warp: kMixSlots source slots (slot 0 doubles as the bank-padded sum
// slice once the bucket's sources are summed) and two tap-row buffers; per
// CTA: the group's bucket tables, sources as 64-bit row offsets.
__host__ __device__ inline MixLayout mix_layout(int KWIN, int tap_stride, int bpg, int group_srcs) {
  MixLayout L{};
  const int slice = 32 * kR + KWIN;
  const int v4 = (slice / 4 + 31) / 32;
  const int lanes = 4 * 32 * v4;  // lane-column layout of a slot
  L.slot_floats = ((padded_len(slice) > lanes ? padded_len(slice) : lanes) + 31) & ~31;
  L.slot_off = 0;  // [SLOTS][slot_floats]
  int off = kMixSlots * L.slot_floats;
  L.taps_off = off;  // [2 buffers][tap_stride] int4 ear pairs
  off += 2 * 4 * tap_stride;
  L.warp_floats = (off + 31) & ~31;
  off = kWarps * L.warp_floats;
  L.boff_off = off;  // [group_srcs] int64
  off += 2 * group_srcs;
  L.bptr_off = off;
  off += (bpg + 4) & ~3;
  L.bdir_off = off;
  off += (bpg + 3) & ~3;
  L.total_bytes = off * 4;
  return L;
}

template <int KWIN, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_mix(MixArgs a) {
  constexpr int COLS = kR + KWIN;
  constexpr int SLICE = 32 * kR + KWIN;
  constexpr int V4 = (SLICE / 4 + 31) / 32;
  constexpr int SLOTS = kMixSlots;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  const MixLayout L = mix_layout(KWIN, a.tap_stride, a.buckets_per_group, a.group_srcs);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* wb = smem + warp * L.warp_floats;
  float* s_slots = wb + L.slot_off;
  float* s_slice = s_slots;  // slot 0 after the sum
  int4* s_taps = reinterpret_cast<int4*>(wb + L.taps_off);  // [2 buffers][tap_stride] ear pairs
  long long* s_boff = reinterpret_cast<long long*>(smem + L.boff_off);
  int* s_bptr = reinterpret_cast<int*>(smem + L.bptr_off);
  int* s_bdir = reinterpret_cast<int*>(smem + L.bdir_off);
  const int SF = L.slot_floats;
  if (warp == 0) tmem_alloc<COLS>(&s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);

  // Items in tile-major order (consecutive items walk the groups of one
  // tile), handed out dynamically: thread 0 takes the next item from a global
  // counter, so CTAs finish together whatever their groups' source counts.
  __shared__ long long s_item;
  int tab_grp = -1, gfirst = 0;
  float chk0 = 0.f, chk1 = 0.f;
  for (;;) {
    if (tid == 0) s_item = (long long)atomicAdd(a.work, 1ull);
    __syncthreads();
    const long long item = s_item;
    if (item >= a.n_items) break;
    const int j = (int)(item / a.groups), grp = (int)(item - (long long)j * a.groups);
    const int b0 = grp * a.buckets_per_group, nb = min(a.buckets - b0, a.buckets_per_group);
    if (grp != tab_grp) {  // the group's bucket tables -> shared memory (all warps at this item)
      __syncthreads();
      for (int i = tid; i <= nb; i += kThreads) s_bptr[i] = __ldg(a.bptr + b0 + i);
      for (int i = tid; i < nb; i += kThreads) s_bdir[i] = __ldg(a.bdir + b0 + i);
      gfirst = __ldg(a.bptr + b0);
      const int gn = __ldg(a.bptr + b0 + nb) - gfirst;
      for (int i = tid; i < gn; i += kThreads) s_boff[i] = (long long)__ldg(a.bsrc + gfirst + i) * a.y_pitch;
      __syncthreads();
      tab_grp = grp;
    }
    const long long* boff = s_boff - gfirst;  // row offset of the i-th source in bucket order: boff[i]
    auto src_off = [&](int i) { return boff[i]; };
    const long long T0 = (long long)j * kW;
    const long long w0 = T0 + (long long)warp * 32 * kR - KWIN;  // signal index of s_slice[0]
    const bool interior = w0 >= 0 && w0 + SLICE <= a.T;
    auto prefetch = [&](int k) {  // bucket k's first SLOTS sources (lane columns) and its two tap rows
      const int i0 = s_bptr[k], n = min(s_bptr[k + 1] - i0, SLOTS);
      if (interior) {
        for (int u = 0; u < n; ++u) {
          const float4* ys = reinterpret_cast<const float4*>(a.y + src_off(i0 + u) + w0);
          float4* sl = reinterpret_cast<float4*>(s_slots + u * SF);
#pragma unroll
          for (int q = 0; q < V4; ++q) {
            const int c = lane + 32 * q;
            if (c < SLICE / 4) cp_async16(&sl[c], ys + c);
          }
        }
      }
      const int dir = s_bdir[k];
      int4* tb = s_taps + (k & 1) * a.tap_stride;
      const int4* tg = a.etaps + (long long)dir * a.tap_stride;
      for (int i = lane; i < a.tap_stride; i += 32) cp_async16(tb + i, tg + i);
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
#pragma unroll
        for (int u = 0; u < SLOTS; ++u) {  // all slot loads can issue before the adds
          if (u < n) {
#pragma unroll
            for (int q = 0; q < V4; ++q) {
              const int c = lane + 32 * q;
              if (c < SLICE / 4) {
                const float4 l = reinterpret_cast<const float4*>(s_slots + u * SF)[c];
                fadd2(v[q].x, v[q].y, l.x, l.y);
                fadd2(v[q].z, v[q].w, l.z, l.w);
              }
            }
          }
        }
        for (int i = i0 + SLOTS; i < i1; ++i) {
          const float4* ys = reinterpret_cast<const float4*>(a.y + src_off(i) + w0);
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
          const float* ys = a.y + src_off(i);
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
      __syncwarp();  // every lane's slot reads are done: slot 0 takes the sum; tap rows of k visible
      {
        float* sb = s_slice + padi(4 * lane);  // padi(4*(lane + 32q)) = padi(4*lane) + 144q
#pragma unroll
        for (int q = 0; q < V4; ++q)
          if (lane + 32 * q < SLICE / 4) *reinterpret_cast<float4*>(sb + 144 * q) = v[q];
      }
      __syncwarp();
      const int4* tp = s_taps + (k & 1) * a.tap_stride;
      const int dir = s_bdir[k];
      {
#pragma unroll
        for (int c = 0; c < COLS; c += 16) {
          // 16 | (16 * lane + c), so padi(16 * lane + c + 4q) = padi(16 * lane + c) + 4q
          const float4* row = reinterpret_cast<const float4*>(&s_slice[padi(16 * lane + c)]);
          float w[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t4 = row[q];
            w[4 * q] = t4.x;
            w[4 * q + 1] = t4.y;
            w[4 * q + 2] = t4.z;
            w[4 * q + 3] = t4.w;
          }
          tmem_st16_nb(tlane + c, w);
        }
        tmem_wait_st();
      }
      __syncwarp();                     // the slice (slot 0) has been read
      if (k + 1 < nb) prefetch(k + 1);  // next bucket's loads overlap this bucket's taps
      const float keepB = a.ears > 1 ? 1.f : 0.f;
      if constexpr (NNZT > 0) {
        float XA0[16], XB0[16], XA1[16], XB1[16];
        int4 t = tp[0];
        int4 tn = tp[NNZT > 1 ? 1 : 0];
        tmem_ld16(XA0, tlane + t.x);
        tmem_ld16(XB0, tlane + t.z);
#pragma unroll
        for (int kk = 0; kk < NNZT; ++kk) {
          const int4 tnn = tp[kk + 2 < NNZT ? kk + 2 : NNZT - 1];
          float(&XA)[16] = (kk & 1) ? XA1 : XA0;
          float(&XB)[16] = (kk & 1) ? XB1 : XB0;
          float(&YA)[16] = (kk & 1) ? XA0 : XA1;
          float(&YB)[16] = (kk & 1) ? XB0 : XB1;
          const unsigned na = tlane + tn.x, nb2 = tlane + tn.z;
          tmem_wait_ld();
          if (kk + 1 < NNZT) {
            tmem_ld16(YA, na);
            tmem_ld16(YB, nb2);
          }
          const float va = __int_as_float(t.y), vb = __int_as_float(t.w) * keepB;
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
          t = tn;
          tn = tnn;
        }
      } else {
        const int nA = __ldg(a.row_nnz + dir);
        const int nB = a.ears > 1 ? __ldg(a.row_nnz + a.dirs + dir) : 0;
        const int nk = max(nA, nB);
        for (int kk = 0; kk < nk; ++kk) {
          const int4 t = tp[kk];
          float XA[16], XB[16];
          tmem_ld16(XA, tlane + t.x);
          tmem_ld16(XB, tlane + t.z);
          tmem_wait_ld();
          const float va = kk < nA ? __int_as_float(t.y) : 0.f;
          const float vb = kk < nB ? __int_as_float(t.w) : 0.f;
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
    __syncthreads();  // s_item is rewritten for the next item
  }
  cp_async_wait_all();
  const bool bad = !isfinite(chk0 + chk1);
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<COLS>(s_tbase);
}

template <int KWIN, int NNZT>
static cudaError_t launch_mix_t(const MixArgs& a, int sm_count, cudaStream_t st) {
  const int bytes = mix_layout(KWIN, a.tap_stride, a.buckets_per_group, a.group_srcs).total_bytes;
  auto kern = k_mix<KWIN, NNZT>;
  cudaError_t err = ensure_smem(reinterpret_cast<const void*>(kern), bytes);
  if (err != cudaSuccess) return err;
  // co-resident CTAs: TMEM allows 512 / COLS, shared memory may allow fewer
  int dev = 0, smem_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess)
    smem_sm = 228 * 1024;
  const int per_sm = std::max(1, std::min(512 / (kR + KWIN), smem_sm / (bytes + 2048)));  // + static + reserved
  long long grid = (long long)sm_count * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, bytes, st>>>(a);
  return cudaGetLastError();
}

template <int KWIN>
static cudaError_t mix_nnz(const MixArgs& a, int nnz_uniform, int sm, cudaStream_t st) {
  switch (nnz_uniform) {
    case 8: return launch_mix_t<KWIN, 8>(a, sm, st);
    case 16: return launch_mix_t<KWIN, 16>(a, sm, st);
    case 24: return launch_mix_t<KWIN, 24>(a, sm, st);
    case 32: return launch_mix_t<KWIN, 32>(a, sm, st);
    default: return launch_mix_t<KWIN, 0>(a, sm, st);
  }
}

cudaError_t launch_mix(const MixArgs& a, int kwin, int nnz_uniform, int sm_count, cudaStream_t st) {
  switch (kwin) {
    case 112: return mix_nnz<112>(a, nnz_uniform, sm_count, st);
    case 240: return mix_nnz<240>(a, nnz_uniform, sm_count, st);
    case 496: return mix_nnz<496>(a, nnz_uniform, sm_count, st);
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
// Two kernels; k_stream_cl (below, clusters of kStreamCL CTAs exchanging
// partials through distributed shared memory) is the default, k_stream_step
// (two global ticketed levels) the TOEP_STREAM_CLUSTER=0 alternative.
// k_stream_step: one launch per block of B <= 256 samples (latency path).  CTA c owns
// src_per_cta sources; thread t owns output sample t for both ears.  The CTA
// loads its sources' [history | block] windows and tap rows into shared
// memory in one vectorised round, accumulates per-thread (3 instructions per
// tap: broadcast tap, window sample, FFMA), writes one partial and rolls the
// sources' history.  Partials are reduced deterministically in two ticketed
// levels (groups of kStreamGroup CTAs, then the groups), and the very last CTA
// applies f_e over [z history | z block] and rolls the z history.
// shared-memory tap-row pitch of k_stream_step (rows read 8 taps at a time)
__host__ __device__ inline int stream_tap_pitch(int tap_stride) { return (tap_stride + 7) / 8 * 8; }


__device__ __forceinline__ bool stream_last_arrival(unsigned int* ticket, unsigned int n) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == n - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

#ifndef TOEP_STREAM_PROF
#define TOEP_STREAM_PROF 0
#endif
#if TOEP_STREAM_PROF
__device__ unsigned long long g_sprof[8];
__device__ unsigned g_sprof_n;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SPROF(i) \
  if (threadIdx.x == 0) atomicMax(&g_sprof[i], gtime())
#else
#define SPROF(i)
#endif

__global__ void __launch_bounds__(256) k_stream_step(StreamArgs a) {
  extern __shared__ __align__(16) float sm[];
#if TOEP_STREAM_PROF
  if (threadIdx.x == 0) atomicMin(&g_sprof[0], gtime());
#endif
  const int tid = threadIdx.x;
  const int L = a.H + a.B;  // multiple of 4 (host checks)
  const int s0 = blockIdx.x * a.src_per_cta;
  const int ns = min(a.S - s0, a.src_per_cta);
  const int tsp = stream_tap_pitch(a.tap_stride);
  float* s_w = sm;                                                // [ns][L]
  int2* s_tap = reinterpret_cast<int2*>(sm + a.src_per_cta * L);  // [ns][ears][tsp] (zero-padded rows)
  int* s_nnz = reinterpret_cast<int*>(s_tap + a.src_per_cta * a.ears * tsp);
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
    // this CTA's sources' tap rows are contiguous in the per-source table;
    // shared rows padded to tsp (a multiple of 8) with zero taps
    const int2* st = a.src_taps + (long long)s0 * a.ears * a.tap_stride;
    for (int i = tid; i < ns * a.ears * tsp; i += blockDim.x) {
      const int row = i / tsp, k = i - row * tsp;
      s_tap[i] = k < a.tap_stride ? __ldg(st + (long long)row * a.tap_stride + k) : make_int2(0, 0);
    }
    for (int i = tid; i < ns * a.ears; i += blockDim.x) s_nnz[i] = __ldg(a.src_nnz + (long long)s0 * a.ears + i);
  }
  __syncthreads();
  SPROF(1);
  const int t = tid;
  float acc0 = 0.f, acc1 = 0.f;
  if (t < a.B) {
    // taps 8 at a time: the 8 (offset, value) pairs by four broadcast 16-byte
    // loads, then 8 independent window loads (no load waits on another), two
    // accumulators per ear (even / odd taps)
    float acc0b = 0.f, acc1b = 0.f;
    for (int s = 0; s < ns; ++s) {
      const float* w = s_w + s * L + a.H + t;
      for (int e = 0; e < a.ears; ++e) {
        const int2* tr = s_tap + (s * a.ears + e) * tsp;
        const int n = s_nnz[s * a.ears + e];
        float ea = 0.f, eb = 0.f;
        for (int k0 = 0; k0 < n; k0 += 8) {
          int2 tp[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int4 v = *reinterpret_cast<const int4*>(tr + k0 + 2 * q);
            tp[2 * q] = make_int2(v.x, v.y);
            tp[2 * q + 1] = make_int2(v.z, v.w);
          }
          float wv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) wv[q] = w[-tp[q].x];  // padding taps: offset 0, value 0
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            ea = fmaf(__int_as_float(tp[q].y), wv[q], ea);
            eb = fmaf(__int_as_float(tp[q + 1].y), wv[q + 1], eb);
          }
        }
        if (e == 0) {
          acc0 += ea;
          acc0b += eb;
        } else {
          acc1 += ea;
          acc1b += eb;
        }
      }
    }
    acc0 += acc0b;
    acc1 += acc1b;
    a.part[((long long)blockIdx.x * a.ears) * a.B + t] = acc0;
    if (a.ears > 1) a.part[((long long)blockIdx.x * a.ears + 1) * a.B + t] = acc1;
  }
  SPROF(2);
  if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && (tid & 31) == 0) atomicOr(a.nonfinite, 1);
  // roll the sources' history: keep the last H samples of [hist | block]
  for (int i = tid; i < ns * (a.H / 4); i += blockDim.x) {
    const int s = i / (a.H / 4), q = i - s * (a.H / 4);
    *reinterpret_cast<float4*>(a.yhist + (long long)(s0 + s) * a.H + 4 * q) =
        *reinterpret_cast<const float4*>(&s_w[s * L + a.B + 4 * q]);
  }
  // ---- level 1: the last CTA of each group sums the group's partials and
  //      applies f over [group z history | group z block] (f is linear, so
  //      out = sum over groups of f * z_g; each group keeps its own z history)
  const int groups = (gridDim.x + kStreamGroup - 1) / kStreamGroup;
  const int grp = blockIdx.x / kStreamGroup;
  const int c0 = grp * kStreamGroup, nc = min((int)gridDim.x - c0, kStreamGroup);
  SPROF(3);
  if (!stream_last_arrival(a.ticket + grp, nc)) return;
  SPROF(4);
  const long long cs = (long long)a.ears * a.B;
  float* s_z = sm;                          // [ears][zh + B]
  float* s_f = sm + a.ears * (a.zh + a.B);  // [ears][lf_pad]
  float* zh_g = a.zhist + (long long)grp * a.ears * a.zh;
  // every load of this level is issued before any is used (one memory latency):
  // the group's partials of this thread's two outputs (ears x B <= 2 x 256), z history, f
  const int nout = a.ears * a.B;
  float zp[2][kStreamGroup];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = tid + h * 256;
#pragma unroll
    for (int u = 0; u < kStreamGroup; ++u) zp[h][u] = (i < nout && u < nc) ? __ldcg(a.part + (c0 + u) * cs + i) : 0.f;
  }
  for (int i = tid; i < a.ears * a.zh; i += blockDim.x) {
    const int e = i / a.zh, k = i - e * a.zh;
    s_z[e * (a.zh + a.B) + k] = zh_g[i];
  }
  for (int i = tid; i < a.ears * a.lf_pad; i += blockDim.x) s_f[i] = __ldg(a.f + i);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = tid + h * 256;
#pragma unroll
    for (int w = kStreamGroup / 2; w > 0; w /= 2)
#pragma unroll
      for (int u = 0; u < w; ++u) zp[h][u] += zp[h][u + w];
    if (i < nout) {
      const int e = i / a.B, tt = i - e * a.B;
      s_z[e * (a.zh + a.B) + a.zh + tt] = zp[h][0];
    }
  }
  __syncthreads();
#if TOEP_STREAM_PROF
  if (tid == 0) g_sprof[7] = gtime();
#endif
  // f over [z history | z block]: a thread takes 4 consecutive outputs of one
  // ear and slides a 4-sample register window down the taps (one shared load
  // per tap for 4 FMAs, f 4 taps per load); shared-load bandwidth, not FMA,
  // bounded the one-output-per-thread form
  for (int u = tid; u < nout / 4; u += blockDim.x) {
    const int e = u / (a.B / 4), tt = 4 * (u - e * (a.B / 4));
    const float* z = s_z + e * (a.zh + a.B) + a.zh + tt;
    const float* ff = s_f + e * a.lf_pad;
    float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
    float x0 = z[0], x1 = z[1], x2 = z[2], x3 = z[3];  // x_k = z[tt + k - jj]
#pragma unroll 2
    for (int jj = 0; jj < a.lf_pad; jj += 4) {
      const float4 f4 = *reinterpret_cast<const float4*>(ff + jj);
#define TOEP_FTAP(fv, next)                                                                   \
  o0 = fmaf(fv, x0, o0);                                                                      \
  o1 = fmaf(fv, x1, o1);                                                                      \
  o2 = fmaf(fv, x2, o2);                                                                      \
  o3 = fmaf(fv, x3, o3);                                                                      \
  x3 = x2;                                                                                    \
  x2 = x1;                                                                                    \
  x1 = x0;                                                                                    \
  x0 = z[next];
      TOEP_FTAP(f4.x, -jj - 1)
      TOEP_FTAP(f4.y, -jj - 2)
      TOEP_FTAP(f4.z, -jj - 3)
      TOEP_FTAP(f4.w, -jj - 4)
#undef TOEP_FTAP
    }
    float* gp = a.gpart + grp * cs + (long long)e * a.B + tt;
    *reinterpret_cast<float4*>(gp) = make_float4(o0, o1, o2, o3);
  }
  __syncthreads();
  for (int i = tid; i < a.ears * a.zh; i += blockDim.x) {
    const int e = i / a.zh, k = i - e * a.zh;
    zh_g[i] = s_z[e * (a.zh + a.B) + a.B + k];
  }
  if (tid == 0) a.ticket[grp] = 0u;
  SPROF(5);
  // ---- level 2: the last group sums the groups' filtered blocks (fixed order)
  if (!stream_last_arrival(a.ticket + groups, groups)) return;
  SPROF(6);
  for (int i = tid; i < a.ears * a.B; i += blockDim.x) {
    const int e = i / a.B, tt = i - e * a.B;
    float o = 0.f;
    for (int g = 0; g < groups; ++g) o += __ldcg(a.gpart + g * cs + i);
    a.out[(long long)e * a.out_pitch + tt] = o;
  }
  if (tid == 0) a.ticket[groups] = 0u;
#if TOEP_STREAM_PROF
  __syncthreads();
  if (tid == 0) {
    const unsigned long long t7 = gtime(), t0 = g_sprof[0];
    printf("sprof ns: load %llu compute %llu roll+partial %llu l1wait %llu l1sum(last grp) %llu l1 %llu l2wait %llu l2 %llu\n",
           g_sprof[1] - t0, g_sprof[2] - t0, g_sprof[3] - t0, g_sprof[4] - t0, g_sprof[7] - t0, g_sprof[5] - t0,
           g_sprof[6] - t0, t7 - t0);
    g_sprof[0] = ~0ull;
    for (int i = 1; i < 8; ++i) g_sprof[i] = 0;
  }
#endif
}

// ---- cluster variant (the default): the CTAs of a cluster of kStreamCL
// exchange their partials through distributed shared memory instead of a
// global ticket level, and every CTA of the cluster applies f to its own
// slice of the block (the one-CTA-per-group f was the longest phase); the
// clusters meet in one ticketed level per slice.  Same per-CTA source work as
// k_stream_step; sums in fixed order (deterministic).
__device__ __forceinline__ unsigned stream_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void stream_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_map(unsigned cta_addr, unsigned rank) {
  unsigned r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(cta_addr), "r"(rank));
  return r;
}
// plain (non-volatile) so the kStreamCL loads of a sum are issued back to back
__device__ __forceinline__ float ld_cluster_f32(unsigned cluster_addr) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cluster_addr));
  return v;
}
// sum over the cluster's CTAs (rank order) of the float at this CTA-relative shared address
__device__ __forceinline__ float sum_cluster_f32(const unsigned (&base)[kStreamCL], unsigned off) {
  float x[kStreamCL];
#pragma unroll
  for (int r = 0; r < kStreamCL; ++r) x[r] = ld_cluster_f32(base[r] + off);
  float v = 0.f;
#pragma unroll
  for (int r = 0; r < kStreamCL; ++r) v += x[r];
  return v;
}

// k_stream_cl shared memory (floats): the per-CTA load area (windows, taps),
// then the exchange inbox, summed window, f and the owner's old history
__host__ __device__ inline int stream_cl_inbox_off(const StreamArgs& a) {
  const int per_cta = a.src_per_cta * (a.H + a.B) + a.src_per_cta * a.ears * stream_tap_pitch(a.tap_stride) * 2 +
                      a.src_per_cta * a.ears;
  return (per_cta + 3) & ~3;
}
__host__ __device__ inline size_t stream_cl_smem_floats(const StreamArgs& a) {
  const int SL = (a.B + kStreamCL - 1) / kStreamCL, ZW = a.lf_pad - 1 + SL;
  return (size_t)stream_cl_inbox_off(a) + (size_t)kStreamCL * a.ears * ZW + (size_t)((a.ears * ZW + 3) & ~3) +
         (size_t)a.ears * a.lf_pad + (size_t)a.ears * a.zh;
}

__global__ void __launch_bounds__(256) k_stream_cl(StreamArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
#if TOEP_STREAM_PROF
  if (threadIdx.x == 0) atomicMin(&g_sprof[0], gtime());
#endif
  const int L = a.H + a.B;
  const int crank = (int)stream_ctarank(), cl = blockIdx.x / kStreamCL, ncl = gridDim.x / kStreamCL;
  const int s0 = blockIdx.x * a.src_per_cta;
  const int ns = max(0, min(a.S - s0, a.src_per_cta));
  // every CTA of the cluster has started before any stores into its shared
  // memory (waited for just before the exchange)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int tsp = stream_tap_pitch(a.tap_stride);
  float* s_w = sm;
  int2* s_tap = reinterpret_cast<int2*>(sm + a.src_per_cta * L);
  int* s_nnz = reinterpret_cast<int*>(s_tap + a.src_per_cta * a.ears * tsp);
  float chk = 0.f;
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
    const int2* st = a.src_taps + (long long)s0 * a.ears * a.tap_stride;
    for (int i = tid; i < ns * a.ears * tsp; i += blockDim.x) {
      const int row = i / tsp, k = i - row * tsp;
      s_tap[i] = k < a.tap_stride ? __ldg(st + (long long)row * a.tap_stride + k) : make_int2(0, 0);
    }
    for (int i = tid; i < ns * a.ears; i += blockDim.x) s_nnz[i] = __ldg(a.src_nnz + (long long)s0 * a.ears + i);
  }
  __syncthreads();
  const int t = tid;
  float acc0 = 0.f, acc1 = 0.f;
  if (t < a.B) {
    float acc0b = 0.f, acc1b = 0.f;
    for (int s = 0; s < ns; ++s) {
      const float* w = s_w + s * L + a.H + t;
      for (int e = 0; e < a.ears; ++e) {
        const int2* tr = s_tap + (s * a.ears + e) * tsp;
        const int n = s_nnz[s * a.ears + e];
        float ea = 0.f, eb = 0.f;
        for (int k0 = 0; k0 < n; k0 += 8) {
          int2 tp[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int4 v = *reinterpret_cast<const int4*>(tr + k0 + 2 * q);
            tp[2 * q] = make_int2(v.x, v.y);
            tp[2 * q + 1] = make_int2(v.z, v.w);
          }
          float wv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) wv[q] = w[-tp[q].x];
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            ea = fmaf(__int_as_float(tp[q].y), wv[q], ea);
            eb = fmaf(__int_as_float(tp[q + 1].y), wv[q + 1], eb);
          }
        }
        if (e == 0) {
          acc0 += ea;
          acc0b += eb;
        } else {
          acc1 += ea;
          acc1b += eb;
        }
      }
    }
    acc0 += acc0b;
    acc1 += acc1b;
  }
  if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && (tid & 31) == 0) atomicOr(a.nonfinite, 1);
  for (int i = tid; i < ns * (a.H / 4); i += blockDim.x) {
    const int s = i / (a.H / 4), q = i - s * (a.H / 4);
    *reinterpret_cast<float4*>(a.yhist + (long long)(s0 + s) * a.H + 4 * q) =
        *reinterpret_cast<const float4*>(&s_w[s * L + a.B + 4 * q]);
  }
  // ---- exchange (push): CTA c owns the block slice [p0_c, p1_c) and needs z
  //      over its window [p0_c - (lf_pad - 1), p1_c); every CTA stores its
  //      partial's samples of each window into the owner's inbox slot for its
  //      rank (remote shared-memory stores, no round trips), then one cluster
  //      barrier; the z history the window needs is read before the barrier,
  //      so the owner of the block's last sample may overwrite it after
  const int SL = (a.B + kStreamCL - 1) / kStreamCL;
  const int ZW = a.lf_pad - 1 + SL;                    // window per ear
  const int p0 = min(a.B, crank * SL), p1 = min(a.B, p0 + SL);
  const int w0 = p0 - (a.lf_pad - 1);                  // window start (may be < 0: history)
  float* s_in = sm + stream_cl_inbox_off(a);           // [kStreamCL][ears][ZW] partials by source rank
  float* s_zl = s_in + kStreamCL * a.ears * ZW;        // [ears][ZW] summed window
  float* s_f = s_zl + ((a.ears * ZW + 3) & ~3);        // [ears][lf_pad]
  const float* zh_c = a.zhist + (long long)cl * a.ears * a.zh;
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  if (t < a.B) {
    const unsigned my_in = (unsigned)__cvta_generic_to_shared(s_in) + 4u * (unsigned)(crank * a.ears * ZW);
#pragma unroll
    for (int c = 0; c < kStreamCL; ++c) {
      const int k = t - (min(a.B, c * SL) - (a.lf_pad - 1));  // t in CTA c's window
      if (k >= 0 && k < ZW && min(a.B, c * SL) < a.B && t < min(a.B, min(a.B, c * SL) + SL)) {
        const unsigned dst = cluster_map(my_in + 4u * (unsigned)k, (unsigned)c);
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(acc0) : "memory");
        if (a.ears > 1)
          asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst + 4u * (unsigned)ZW), "f"(acc1) : "memory");
      }
    }
  }
  for (int i = tid; i < a.ears * ZW; i += blockDim.x) {  // history part of the window
    const int e = i / ZW, k = i - e * ZW;
    const int q = w0 + k;
    if (q < 0) s_zl[i] = zh_c[e * a.zh + a.zh + q];
  }
  for (int i = tid; i < a.ears * a.lf_pad; i += blockDim.x) s_f[i] = __ldg(a.f + i);
  const int owner = (a.B - 1) / SL;  // holds position B - 1: writes the next z history
  float* s_zo = s_f + a.ears * a.lf_pad;  // [ears][zh] old history (owner, when B < zh)
  if (crank == owner && a.B < a.zh)
    for (int i = tid; i < a.ears * a.zh; i += blockDim.x) s_zo[i] = zh_c[i];
  SPROF(1);
  stream_cluster_sync();
  SPROF(2);
  for (int i = tid; i < a.ears * ZW; i += blockDim.x) {
    const int e = i / ZW, k = i - e * ZW;
    const int q = w0 + k;
    if (q >= 0) {
      float v = 0.f;
      if (q < p1) {
#pragma unroll
        for (int r = 0; r < kStreamCL; ++r) v += s_in[(r * a.ears + e) * ZW + k];
      }
      s_zl[i] = v;
    }
  }
  __syncthreads();
  SPROF(3);
  if (crank == owner) {  // next history: the last zh samples of [z history | z block]
    for (int i = tid; i < a.ears * a.zh; i += blockDim.x) {
      const int e = i / a.zh, k = i - e * a.zh;
      const int q = a.B + k - a.zh;  // block position (< 0: old history)
      a.zhist[(long long)cl * a.ears * a.zh + i] = q < 0 ? s_zo[e * a.zh + a.zh + q] : s_zl[e * ZW + (q - w0)];
    }
  }
  const long long cs = (long long)a.ears * a.B;
  for (int i = tid; i < a.ears * (p1 - p0); i += blockDim.x) {
    const int e = i / (p1 - p0), p = p0 + (i - e * (p1 - p0));
    const float* z = s_zl + e * ZW + (p - w0);
    const float* ff = s_f + e * a.lf_pad;
    float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;  // lf_pad is a multiple of 16
#pragma unroll 2
    for (int jj = 0; jj < a.lf_pad; jj += 4) {
      o0 = fmaf(ff[jj], z[-jj], o0);
      o1 = fmaf(ff[jj + 1], z[-jj - 1], o1);
      o2 = fmaf(ff[jj + 2], z[-jj - 2], o2);
      o3 = fmaf(ff[jj + 3], z[-jj - 3], o3);
    }
    const float o = (o0 + o1) + (o2 + o3);
    if (ncl == 1) a.out[(long long)e * a.out_pitch + p] = o;
    else a.gpart[cl * cs + (long long)e * a.B + p] = o;
  }
  SPROF(4);
  SPROF(5);
  if (ncl == 1) return;
  // ---- across clusters: the last cluster to finish this slice sums it (fixed order)
  if (!stream_last_arrival(a.ticket + crank, (unsigned)ncl)) return;
  SPROF(6);
  for (int i = tid; i < a.ears * (p1 - p0); i += blockDim.x) {
    const int e = i / (p1 - p0), p = p0 + (i - e * (p1 - p0));
    const float* g = a.gpart + (long long)e * a.B + p;
    float o = 0.f;
    int c = 0;
    for (; c + 8 <= ncl; c += 8) {  // 8 independent loads, then the adds in order
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcg(g + (c + u) * cs);
#pragma unroll
      for (int u = 0; u < 8; ++u) o += x[u];
    }
    for (; c < ncl; ++c) o += __ldcg(g + c * cs);
    a.out[(long long)e * a.out_pitch + p] = o;
  }
  if (tid == 0) a.ticket[crank] = 0u;
#if TOEP_STREAM_PROF
  SPROF(7);
  if (tid == 0 && atomicAdd(&g_sprof_n, 1u) == kStreamCL - 1) {  // the last slice to finish prints
    const unsigned long long t0 = g_sprof[0];
    printf("sprof-cl ns: partial %llu bar1 %llu zgather %llu f %llu bar2 %llu l2wait %llu end %llu\n",
           g_sprof[1] - t0, g_sprof[2] - t0, g_sprof[3] - t0, g_sprof[4] - t0, g_sprof[5] - t0, g_sprof[6] - t0,
           g_sprof[7] - t0);
    g_sprof[0] = ~0ull;
    for (int i = 1; i < 8; ++i) g_sprof[i] = 0;
    g_sprof_n = 0;
  }
#endif
}

__global__ void k_stream_gather_taps(const int2* __restrict__ raw, const int* __restrict__ nnz,
                                     const int* __restrict__ src_dir, int S, int ears, int dirs, int stride,
                                     int2* __restrict__ out, int* __restrict__ out_nnz) {
  const long long total = (long long)S * ears * stride;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long se = i / stride;
    const int k = (int)(i - se * stride);
    const int s = (int)(se / ears), e = (int)(se - (long long)s * ears);
    const long long row = (long long)e * dirs + src_dir[s];
    out[i] = raw[row * stride + k];
    if (k == 0) out_nnz[se] = nnz[row];
  }
}

cudaError_t launch_stream_gather_taps(const int2* raw, const int* nnz, const int* src_dir, int S, int ears, int dirs,
                                      int stride, int2* out, int* out_nnz, cudaStream_t st) {
  const long long total = (long long)S * ears * stride;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 1024);
  k_stream_gather_taps<<<std::max(blocks, 1), 256, 0, st>>>(raw, nnz, src_dir, S, ears, dirs, stride, out, out_nnz);
  return cudaGetLastError();
}

// TOEP_STREAM_CLUSTER=0 selects the two-level ticketed kernel (A/B runs;
// read once per streamer, at creation)
bool stream_cluster_enabled() {
  const char* ev = getenv("TOEP_STREAM_CLUSTER");
  return !(ev && atoi(ev) == 0);
}

int stream_ctas(int S, int spc, bool cluster) {
  const int c = (S + spc - 1) / spc;
  return cluster ? (c + kStreamCL - 1) / kStreamCL * kStreamCL : c;
}

cudaError_t launch_stream_step(const StreamArgs& a, cudaStream_t st) {
  const size_t per_cta = (size_t)a.src_per_cta * (a.H + a.B) +
                         (size_t)a.src_per_cta * a.ears * stream_tap_pitch(a.tap_stride) * 2 +
                         (size_t)a.src_per_cta * a.ears;
  if (a.cluster) {
    const size_t smem = stream_cl_smem_floats(a) * 4;
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k_stream_cl), (int)smem);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kStreamCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)a.ctas);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_stream_cl, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  const size_t fin = (size_t)a.ears * (a.zh + a.B + a.lf_pad);
  const size_t smem = std::max(per_cta, fin) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(k_stream_step), (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_stream_step<<<a.ctas, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace toep
