// Fused two-stage renderer: out[e][d] = (y * f_e) * g_{e,d}   (full linear convolution)
//
// Reference semantics: toepnmf Renderer.render (pkg/src/toepnmf/engine/__init__.py:238-260)
// = conv_dense(y, f) (_kernels.pyx:11-25) followed by conv_sparse(yf, idx, vals, K)
// (_kernels.pyx:28-44), batched here over every (ear, direction) row of a model.
//
// Layout / schedule:
//   * work item = (ear e, direction group g, time tile j); tile = 2048 outputs,
//     4 warps x 32 lanes x 16 consecutive outputs per lane.
//   * persistent CTAs walk a contiguous range of items, so consecutive items
//     share the ear/group: tap tables stay in shared memory and the resonance
//     halo of the previous tile is reused.
//   * stage 1 (dense resonance FIR, Lf taps) is computed per tile into shared
//     memory with a 16x16 register-blocked FFMA micro-kernel; the intermediate
//     y*f never goes to HBM.
//   * stage 2: each lane writes its (16 + KWIN)-sample window of y*f into its
//     TMEM lane row once per tile; every sparse tap (runtime offset o, weight v)
//     then costs one tcgen05.ld.32x32b.x16 at column KWIN-o plus 16 FFMA.
//   * each warp's 512 outputs per row leave through a cp.async.bulk store.
#include "common.cuh"
#include "launch.h"

namespace toep {

template <int KWIN>
struct RenderCfg {
  static constexpr int COLS = kR + KWIN;     // TMEM columns per lane (power of two)
  static constexpr int YH = KWIN + kR;       // y*f halo kept in front of a tile
  static_assert((COLS & (COLS - 1)) == 0 && COLS >= 32 && COLS <= 512, "TMEM allocation");
  static constexpr int kStageSlots = 2;
};

struct SmemLayout {
  int x_off, f_off, yf_off, stage_off, taps_off, nnz_off, total;
};

__host__ __device__ inline SmemLayout render_smem_layout(int KWIN, bool stage1, int lf_pad, int dpg,
                                                         int tap_stride) {
  SmemLayout L{};
  const int YH = KWIN + kR;
  int off = 0;
  L.x_off = off;
  if (stage1) off += padded_len(kW + YH + lf_pad);
  off = (off + 31) & ~31;
  L.f_off = off;
  if (stage1) off += lf_pad;
  off = (off + 31) & ~31;
  L.yf_off = off;
  off += kW + YH;
  off = (off + 31) & ~31;
  L.stage_off = off;
  off += kWarps * 2 * 32 * kR;
  L.taps_off = off;  // int2 entries (8 B) -> counted in floats x2
  off += 2 * dpg * tap_stride;
  L.nnz_off = off;
  off += dpg;
  L.total = off * 4 + 16;
  return L;
}

template <int KWIN, bool STAGE1, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_render(RenderArgs a) {
  using C = RenderCfg<KWIN>;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  __shared__ long long s_prev_item;

  const SmemLayout L = render_smem_layout(KWIN, STAGE1, a.lf_pad, a.dirs_per_group, a.tap_stride);
  float* s_x = smem + L.x_off;
  float* s_f = smem + L.f_off;
  float* s_yf = smem + L.yf_off;
  float* s_stage = smem + L.stage_off;
  int2* s_taps = reinterpret_cast<int2*>(smem + L.taps_off);
  int* s_nnz = reinterpret_cast<int*>(smem + L.nnz_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tmem_alloc<C::COLS>(&s_tbase);
  if (tid == 0) s_prev_item = -2;
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);

  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);
  int cur_group = -1, cur_ear = -1;
  int slot = 0;
  float* my_stage = s_stage + warp * 2 * 32 * kR;

  for (long long item = it0; item < it1; ++item) {
    const int j = (int)(item % a.n_tiles);
    const long long eg = item / a.n_tiles;
    const int g = (int)(eg % a.groups);
    const int e = (int)(eg / a.groups);
    const long long T0 = (long long)j * kW;
    const bool reuse_halo = STAGE1 && (item == s_prev_item + 1) && j > 0;
    const int d_begin = g * a.dirs_per_group;
    const int nd = min(a.dirs_per_group, a.dirs - d_begin);

    __syncthreads();  // previous item fully consumed (TMEM windows, s_yf, s_taps)

    // ---- tap table for (e, g) --------------------------------------------
    if (g != cur_group || e != cur_ear) {
      const long long row0 = (long long)e * a.dirs + d_begin;
      const int n = nd * a.tap_stride;
      const int2* src = a.taps + row0 * a.tap_stride;
      for (int i = tid; i < n; i += kThreads) s_taps[i] = src[i];
      for (int i = tid; i < nd; i += kThreads) s_nnz[i] = a.row_nnz[row0 + i];
      if (STAGE1 && e != cur_ear)
        for (int i = tid; i < a.lf_pad; i += kThreads) s_f[i] = a.f[(long long)e * a.lf_pad + i];
      cur_group = g;
      cur_ear = e;
    }

    // ---- y*f tile [T0 - YH, T0 + kW) -------------------------------------
    if constexpr (STAGE1) {
      const int xlen = kW + C::YH + a.lf_pad;
      const long long xs = T0 - C::YH - a.lf_pad;  // signal index of s_x[0]
      for (int i = tid; i < xlen; i += kThreads) {
        const long long t = xs + i;
        s_x[padi(i)] = (t >= 0 && t < a.nx) ? __ldg(a.x + t) : 0.f;
      }
      if (reuse_halo) {
        // last YH values of the previous tile become this tile's halo
        for (int i = tid; i < C::YH; i += kThreads) s_yf[i] = s_yf[kW + i];
      }
      __syncthreads();
      if (!reuse_halo) {
        for (int c = tid; c < C::YH / 16; c += kThreads) {
          float acc[16];
#pragma unroll
          for (int r = 0; r < 16; ++r) acc[r] = 0.f;
          fir16_block(acc, s_x, a.lf_pad + 16 * c, s_f, a.lf_pad);
#pragma unroll
          for (int r = 0; r < 16; r += 4)
            *reinterpret_cast<float4*>(&s_yf[16 * c + r]) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
        }
      }
      {
        float acc[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = 0.f;
        fir16_block(acc, s_x, C::YH + a.lf_pad + 16 * tid, s_f, a.lf_pad);
#pragma unroll
        for (int r = 0; r < 16; r += 4)
          *reinterpret_cast<float4*>(&s_yf[C::YH + 16 * tid + r]) =
              make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
      }
    } else {
      const float* xe = a.x + (long long)e * a.x_pitch;
      const long long xs = T0 - C::YH;
      for (int i = tid; i < kW + C::YH; i += kThreads) {
        const long long t = xs + i;
        s_yf[i] = (t >= 0 && t < a.nx) ? __ldg(xe + t) : 0.f;
      }
    }
    if (tid == 0) s_prev_item = item;
    __syncthreads();

    // ---- lane windows -> TMEM ------------------------------------------------
    {
      const int wbase = (C::YH - KWIN) + 16 * tid;  // = 16 + 16*tid
#pragma unroll
      for (int c = 0; c < C::COLS; c += 16) {
        float v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 t4 = *reinterpret_cast<const float4*>(&s_yf[wbase + c + 4 * q]);
          v[4 * q] = t4.x;
          v[4 * q + 1] = t4.y;
          v[4 * q + 2] = t4.z;
          v[4 * q + 3] = t4.w;
        }
        tmem_st16(tlane + c, v);
      }
      tmem_wait_st();
    }

    // ---- sparse reflection stage ------------------------------------------
    const long long out_col = T0 + (long long)warp * 32 * kR;
    const int nd_w = (out_col < a.out_len) ? nd : 0;  // warps wholly past the row end store nothing
    for (int dd = 0; dd < nd_w; ++dd) {
      const int2* tp = s_taps + dd * a.tap_stride;
      float acc[16];
      if constexpr (NNZT > 0) {
        float A[16], B[16];
        int2 cur = tp[0];
        tmem_ld16(A, tlane + cur.x);
#pragma unroll
        for (int k = 0; k < NNZT; ++k) {
          const int2 nxt = tp[k + 1 < NNZT ? k + 1 : k];
          tmem_wait_ld();
          float(&X)[16] = (k & 1) ? B : A;
          float(&Y)[16] = (k & 1) ? A : B;
          if (k + 1 < NNZT) tmem_ld16(Y, tlane + nxt.x);
          const float v = __int_as_float(cur.y);
          if (k == 0) {
#pragma unroll
            for (int r = 0; r < 16; ++r) acc[r] = v * X[r];
          } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) acc[r] = fmaf(v, X[r], acc[r]);
          }
          cur = nxt;
        }
      } else {
        const int nnz = s_nnz[dd];
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = 0.f;
        float X[16];
        for (int k = 0; k < nnz; ++k) {
          const int2 cur = tp[k];
          tmem_ld16(X, tlane + cur.x);
          tmem_wait_ld();
          const float v = __int_as_float(cur.y);
#pragma unroll
          for (int r = 0; r < 16; ++r) acc[r] = fmaf(v, X[r], acc[r]);
        }
      }
      // ---- epilogue: registers -> smem slot -> one bulk store per warp --
      float* st = my_stage + slot * 32 * kR;
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 16; r += 4)
        *reinterpret_cast<float4*>(&st[lane * 16 + r]) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      {
        const long long row = (long long)e * a.dirs + d_begin + dd;
        float* dst = a.out + row * a.out_pitch + out_col;
        if (out_col + 32 * kR <= a.out_len) {
          if (lane == 0) bulk_store(dst, st, 32 * kR * 4);
        } else {  // ragged row end: plain stores, nothing past out_len
          for (int i = lane; i < 32 * kR; i += 32)
            if (out_col + i < a.out_len) dst[i] = st[i];
        }
      }
      slot ^= 1;
    }
  }
  if (lane == 0) bulk_wait_all();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::COLS>(s_tbase);
}

// ---------------------------------------------------------------- launch ----
template <int KWIN, bool STAGE1, int NNZT>
static cudaError_t launch_render_t(const RenderArgs& a, int sm_count, cudaStream_t st) {
  using C = RenderCfg<KWIN>;
  const SmemLayout L = render_smem_layout(KWIN, STAGE1, a.lf_pad, a.dirs_per_group, a.tap_stride);
  auto kern = k_render<KWIN, STAGE1, NNZT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
  if (err != cudaSuccess) return err;
  // TMEM bounds co-residency: at most 512 / COLS CTAs per SM.  Shared memory
  // and registers are sized so the hardware never exceeds that.
  const int per_sm = 512 / C::COLS;
  long long grid = (long long)sm_count * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, L.total, st>>>(a);
  return cudaGetLastError();
}

template <int KWIN, bool STAGE1>
static cudaError_t dispatch_nnz(const RenderArgs& a, int sm, cudaStream_t st) {
  if (a.uniform_nnz) {
    switch (a.tap_stride_nnz) {
      case 4: return launch_render_t<KWIN, STAGE1, 4>(a, sm, st);
      case 8: return launch_render_t<KWIN, STAGE1, 8>(a, sm, st);
      case 12: return launch_render_t<KWIN, STAGE1, 12>(a, sm, st);
      case 16: return launch_render_t<KWIN, STAGE1, 16>(a, sm, st);
      case 24: return launch_render_t<KWIN, STAGE1, 24>(a, sm, st);
      case 32: return launch_render_t<KWIN, STAGE1, 32>(a, sm, st);
      default: break;
    }
  }
  return launch_render_t<KWIN, STAGE1, 0>(a, sm, st);
}

int render_kwin_for(int K) {
  if (K <= 113) return 112;
  if (K <= 241) return 240;
  if (K <= 497) return 496;
  return -1;
}

size_t render_smem_bytes(int kwin, bool stage1, int lf_pad, int dpg, int tap_stride) {
  return (size_t)render_smem_layout(kwin, stage1, lf_pad, dpg, tap_stride).total;
}

cudaError_t launch_render(const RenderArgs& a, int kwin, bool stage1, int sm_count, cudaStream_t st) {
  if (stage1) {
    switch (kwin) {
      case 112: return dispatch_nnz<112, true>(a, sm_count, st);
      case 240: return dispatch_nnz<240, true>(a, sm_count, st);
      case 496: return dispatch_nnz<496, true>(a, sm_count, st);
    }
  } else {
    switch (kwin) {
      case 112: return dispatch_nnz<112, false>(a, sm_count, st);
      case 240: return dispatch_nnz<240, false>(a, sm_count, st);
      case 496: return dispatch_nnz<496, false>(a, sm_count, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace toep
