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
#include <algorithm>

#include "common.cuh"
#include "launch.h"

#ifndef TOEP_RENDER_MINB
#define TOEP_RENDER_MINB 4
#endif

namespace toep {

template <int KWIN>
struct RenderCfg {
  static constexpr int COLS = kR + KWIN;     // TMEM columns per lane (power of two)
  static constexpr int YH = KWIN + kR;       // y*f halo kept in front of a tile
  static_assert((COLS & (COLS - 1)) == 0 && COLS >= 32 && COLS <= 512, "TMEM allocation");
  static constexpr int kStageSlots = 2;
};

struct SmemLayout {
  int region_off, x_off, yf_off, halo_off, f_off, ring_off, nnz_off, bars_off, chunk_pairs, total;
};

constexpr int kStageFloatsPerWarp = 4 * 32 * kR;  // 4 directions x 512 outputs
constexpr int kTapRing = 3;                        // tap-chunk buffers streamed by TMA

// Shared memory plan.  The stage-1 input tile (s_x) and the y*f tile (s_yf)
// are only live between an item's start and its TMEM window write, the bulk
// store staging only during its direction loop, so they share one region.
// Reflection taps are not staged per direction group: chunks of direction
// pairs (int4 {colA, vA, colB, vB} per tap, host-interleaved) stream through a
// kTapRing-deep ring by cp.async.bulk, so one work item covers every
// direction of an ear for its time tile.
__host__ __device__ inline SmemLayout render_smem_layout(int KWIN, bool stage1, int lf_pad, int tap_stride) {
  SmemLayout L{};
  const int YH = KWIN + kR;
  L.region_off = 0;
  L.x_off = 0;
  int tile = stage1 ? ((padded_len(kW + YH + lf_pad) + 31) & ~31) : 0;
  L.yf_off = tile;
  tile += kW + YH;
  int region = tile > kWarps * kStageFloatsPerWarp ? tile : kWarps * kStageFloatsPerWarp;
  int off = (region + 31) & ~31;
  L.halo_off = off;
  off += (YH + 31) & ~31;
  L.f_off = off;
  off += (lf_pad + 31) & ~31;
  int cp = 4096 / (tap_stride * 16);  // pairs per chunk: ~4 KB chunks
  if (cp < 1) cp = 1;
  if (cp > 32) cp = 32;
  L.chunk_pairs = cp;
  L.ring_off = off;  // [kTapRing][cp][tap_stride] int4
  off += kTapRing * cp * tap_stride * 4;
  L.nnz_off = off;  // [kTapRing][cp] int4 {nnzA, nnzB, 0, 0}
  off += kTapRing * cp * 4;
  L.bars_off = off;  // full[kTapRing], empty[kTapRing] (uint64)
  off += 4 * kTapRing;
  L.total = off * 4 + 1024;  // + alignment slack for the 1 KB-aligned base
  return L;
}

// Balanced decomposition: work units are (ear, tile, direction); each
// persistent CTA takes a contiguous unit range snapped to even directions
// (pairs are never split between CTAs), so CTAs differ by at most one
// direction pair of one tile.
struct UnitMap {
  int D, n_tiles;
  long long n_units;
  __device__ void decode(long long u, int& e, int& j, int& dd) const {
    const long long per_ear = (long long)D * n_tiles;
    e = (int)(u / per_ear);
    const long long rem = u - (long long)e * per_ear;
    j = (int)(rem / D);
    dd = (int)(rem - (long long)j * D);
  }
  __device__ long long snap(long long u) const {
    if (u >= n_units) return n_units;
    int e, j, dd;
    decode(u, e, j, dd);
    return u - (dd & 1);
  }
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, const float* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tm),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

template <int KWIN, bool STAGE1, int NNZT>
__global__ void __launch_bounds__(kThreads,
                                  (512 / (kR + KWIN)) > 3 ? TOEP_RENDER_MINB : (512 / (kR + KWIN)))
    k_render(RenderArgs a, const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm1) {
  using C = RenderCfg<KWIN>;
  constexpr int NW = kWarps;
  constexpr int NT = 32 * NW;
  extern __shared__ float smem_raw[];
  __shared__ unsigned s_tbase;
  // 1 KB-align the dynamic base by pointer arithmetic on the shared array (keeps the
  // shared address space visible to the compiler: LDS/STS, not generic LD/ST)
  float* smem = smem_raw + (((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) >> 2);

  const SmemLayout L = render_smem_layout(KWIN, STAGE1, a.lf_pad, a.tap_stride);
  float* s_x = smem + L.x_off;
  float* s_yf = smem + L.yf_off;
  float* s_halo = smem + L.halo_off;
  float* s_f = smem + L.f_off;
  int4* s_ring = reinterpret_cast<int4*>(smem + L.ring_off);
  int4* s_rnnz = reinterpret_cast<int4*>(smem + L.nnz_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars_off);
  uint64_t* empty = full + kTapRing;
  const int CP = L.chunk_pairs;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tmem_alloc<C::COLS>(&s_tbase);
  if (tid == 0) {
    for (int i = 0; i < kTapRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    mbar_fence_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const int quarter = warp & 3;
  const unsigned tlane = s_tbase + ((unsigned)(32 * quarter) << 16);

  UnitMap um;
  um.D = a.dirs;
  um.n_tiles = a.n_tiles;
  um.n_units = (long long)a.ears * a.dirs * a.n_tiles;
  const long long u0 = um.snap(um.n_units * blockIdx.x / gridDim.x);
  const long long u1 = um.snap(um.n_units * (blockIdx.x + 1) / gridDim.x);

  int cur_e = -1, prev_j = -2;
  int chunk_base = 0;  // tap chunks consumed by this CTA so far (ring phase bookkeeping)
  float* st = smem + L.region_off + warp * (kStageFloatsPerWarp * kWarps / NW);
  const int half = lane >> 4, inner = (lane & 15) * 16;

  float chk = 0.f;  // x*0 accumulates NaN iff an input sample was inf/NaN (fused DataError check)
  for (long long u = u0; u < u1;) {
    int e, j, dd0;
    um.decode(u, e, j, dd0);
    const int nd = a.dirs;
    const int dd1 = (int)min((long long)nd, dd0 + (u1 - u));
    u += dd1 - dd0;
    const long long T0 = (long long)j * kW;
    const bool reuse_halo = STAGE1 && e == cur_e && (j == prev_j + 1);
    const int p0 = dd0 >> 1, p1 = (dd1 + 1) >> 1;
    const int nchunks = (p1 - p0 + CP - 1) / CP;
    const int4* pairs_e = a.pairs + (long long)e * a.pairs_per_ear * a.tap_stride;
    const int4* pnnz_e = a.pair_nnz + (long long)e * a.pairs_per_ear;
    // tap-chunk producer (warp 0, elected lane): chunk c covers pairs p0 + c*CP ...
    auto issue_chunk = [&](int c) {
      const int g = chunk_base + c;
      const int buf = g % kTapRing;
      mbar_wait(&empty[buf], (unsigned)(((g / kTapRing) & 1) ^ 1));
      const int pb = p0 + c * CP;
      const int np = min(CP, p1 - pb);
      const unsigned bytes_t = (unsigned)(np * a.tap_stride) * 16u;
      mbar_arrive_expect_tx(&full[buf], bytes_t + (unsigned)np * 16u);
      bulk_load(s_ring + buf * CP * a.tap_stride, pairs_e + (long long)pb * a.tap_stride, bytes_t, &full[buf]);
      bulk_load(s_rnnz + buf * CP, pnnz_e + pb, (unsigned)np * 16u, &full[buf]);
    };

    if (lane == 0) bulk_wait_read<0>();  // staging region is about to be reused
    __syncthreads();  // previous item fully consumed (TMEM windows, smem region)
    if (warp == 0 && elect_one())
      for (int c = 0; c < min(kTapRing - 1, nchunks); ++c) issue_chunk(c);
    if (STAGE1 && e != cur_e)
      for (int i = tid; i < a.lf_pad; i += NT) s_f[i] = a.f[(long long)e * a.lf_pad + i];
    cur_e = e;
    prev_j = j;

    // ---- y*f tile [T0 - YH, T0 + kW) -------------------------------------
    if constexpr (STAGE1) {
      const int xlen = kW + C::YH + a.lf_pad;
      const long long xs = T0 - C::YH - a.lf_pad;  // signal index of s_x[0]
      for (int i = tid; i < xlen; i += NT) {
        const long long t = xs + i;
        const float v = (t >= 0 && t < a.nx) ? __ldg(a.x + t) : 0.f;
        chk = fmaf(v, 0.f, chk);
        s_x[padi(i)] = v;
      }
      if (reuse_halo)  // last YH values of the previous tile are this tile's halo
        for (int i = tid; i < C::YH; i += NT) s_yf[i] = s_halo[i];
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
      if (tid < kThreads) {
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
      for (int i = tid; i < kW + C::YH; i += NT) {
        const long long t = xs + i;
        const float v = (t >= 0 && t < a.nx) ? __ldg(xe + t) : 0.f;
        chk = fmaf(v, 0.f, chk);
        s_yf[i] = v;
      }
    }
    __syncthreads();

    // ---- lane windows -> TMEM; keep the next tile's halo -----------------
    {
      const int wbase = (C::YH - KWIN) + 16 * (32 * quarter + lane);  // = 16 + 16*lane row
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
      if (STAGE1)
        for (int i = tid; i < C::YH; i += NT) s_halo[i] = s_yf[kW + i];
      tmem_wait_st();
    }
    __syncthreads();  // s_yf fully read: the region becomes bulk-store staging

    // ---- sparse reflection stage, two directions per pass ------------------
    const long long col = T0 + (long long)quarter * 32 * kR;
    const bool store = col < a.out_len;  // warps wholly past the row end compute but store nothing
    int c = 0, kin = 0, g = chunk_base, buf = chunk_base % kTapRing;  // chunk cursor (no division in the loop)
    for (int p = p0; p < p1; ++p) {
      if (kin == CP) {
        kin = 0;
        ++c;
        ++g;
        buf = (buf + 1 == kTapRing) ? 0 : buf + 1;
      }
      if (kin == 0) {
        if (warp == 0 && c + kTapRing - 1 < nchunks && elect_one()) issue_chunk(c + kTapRing - 1);
        __syncwarp();
        mbar_wait(&full[buf], (unsigned)((g / kTapRing) & 1));
      }
      const int4* tp = s_ring + (buf * CP + kin) * a.tap_stride;
      float accA[16], accB[16];
      if constexpr (NNZT > 0) {
        // software pipeline: the TMEM loads of tap k+1 are in flight while
        // tap k's 32 FFMA issue (tcgen05.wait::ld only ever waits for tap k)
        float XA0[16], XB0[16], XA1[16], XB1[16];
        int4 t = tp[0];
        int4 tn = tp[NNZT > 1 ? 1 : 0];  // taps are read two ahead of their TMEM loads
        tmem_ld16(XA0, tlane + t.x);
        tmem_ld16(XB0, tlane + t.z);
#pragma unroll
        for (int k = 0; k < NNZT; ++k) {
          const int4 tnn = tp[k + 2 < NNZT ? k + 2 : NNZT - 1];
          float(&XA)[16] = (k & 1) ? XA1 : XA0;
          float(&XB)[16] = (k & 1) ? XB1 : XB0;
          float(&YA)[16] = (k & 1) ? XA0 : XA1;
          float(&YB)[16] = (k & 1) ? XB0 : XB1;
          const unsigned na = tlane + tn.x, nb = tlane + tn.z;
          tmem_wait_ld();
          if (k + 1 < NNZT) {
            tmem_ld16(YA, na);
            tmem_ld16(YB, nb);
          }
          const float va = __int_as_float(t.y), vb = __int_as_float(t.w);
          if (k == 0) {
#pragma unroll
            for (int r = 0; r < 16; r += 2) {
              fmul2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
              fmul2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
            }
          } else {
#pragma unroll
            for (int r = 0; r < 16; r += 2) {
              ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
              ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
            }
          }
          t = tn;
          tn = tnn;
        }
      } else {
        const int4 pn = s_rnnz[buf * CP + kin];
        const int nk = max(pn.x, pn.y);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          accA[r] = 0.f;
          accB[r] = 0.f;
        }
        for (int k = 0; k < nk; ++k) {
          const int4 t = tp[k];
          float XA[16], XB[16];
          tmem_ld16(XA, tlane + t.x);
          tmem_ld16(XB, tlane + t.z);
          tmem_wait_ld();
          const float va = __int_as_float(t.y), vb = __int_as_float(t.w);
#pragma unroll
          for (int r = 0; r < 16; r += 2) {
            ffma2(accA[r], accA[r + 1], XA[r], XA[r + 1], va);
            ffma2(accB[r], accB[r + 1], XB[r], XB[r + 1], vb);
          }
        }
      }
      if (kin == CP - 1 || p + 1 == p1) {  // this warp is done with the chunk's taps
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[buf]);
      }
      ++kin;
      if (!store) continue;
      // ---- epilogue: stage 2 pairs (4 rows), then one proxy fence and
      //      TMA tensor stores of [2 rows x 256] boxes (clipped at out_len)
      const int pp = (p - p0) & 1;
      if (pp == 0) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      {
        float* box = st + (pp * 2 + half) * 512;  // [row][256]
#pragma unroll
        for (int r = 0; r < 16; r += 4) {
          *reinterpret_cast<float4*>(&box[inner + r]) = make_float4(accA[r], accA[r + 1], accA[r + 2], accA[r + 3]);
          *reinterpret_cast<float4*>(&box[256 + inner + r]) =
              make_float4(accB[r], accB[r + 1], accB[r + 2], accB[r + 3]);
        }
      }
      if (pp == 1 || p + 1 == p1) {
        fence_proxy_async_smem();
        __syncwarp();
        if (elect_one()) {
          for (int q = 0; q <= pp; ++q) {
            const int pq = p - pp + q;
            const int rowA = e * a.dirs + 2 * pq;
            const CUtensorMap* tm = (2 * pq + 1 < nd) ? &tm2 : &tm1;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (col + 256 * h < a.out_len) tma_store_2d(tm, st + (q * 2 + h) * 512, (int)(col + 256 * h), rowA);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    chunk_base += nchunks;
  }
  if (a.nonfinite && __any_sync(0xffffffffu, !isfinite(chk)) && lane == 0) atomicOr(a.nonfinite, 1);
  if (lane == 0) bulk_wait_all();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::COLS>(s_tbase);
}

// Interleave direction pairs of each segment of `seg` consecutive rows:
// out[s][p][k] = {colA, vA, colB, vB} of rows (2p, 2p+1) of segment s (B padded
// with a zero tap when the segment is odd); out_nnz[s][p] = {nnzA, nnzB, 0, 0}.
__global__ void k_pair_taps(const int2* __restrict__ rows, const int* __restrict__ nnz, int n_seg, int seg,
                            int stride, int kwin, int4* __restrict__ out, int4* __restrict__ out_nnz) {
  const int P = (seg + 1) / 2;
  const long long total = (long long)n_seg * P * stride;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % stride);
    const long long sp = i / stride;
    const int p = (int)(sp % P), s = (int)(sp / P);
    const long long ra = (long long)s * seg + 2 * p, rb = ra + 1;
    const int2 A = rows[ra * stride + k];
    const int2 B = (2 * p + 1 < seg) ? rows[rb * stride + k] : make_int2(kwin, 0);
    out[i] = make_int4(A.x, A.y, B.x, B.y);
    if (k == 0) out_nnz[sp] = make_int4(nnz[ra], (2 * p + 1 < seg) ? nnz[rb] : 0, 0, 0);
  }
}

// Ear-interleaved taps for the mixdown: out[d][k] = {col_e0, v_e0, col_e1, v_e1}
// of rows d and dirs + d (a zero tap at column kwin when there is one ear).
__global__ void k_ear_pair_taps(const int2* __restrict__ rows, int dirs, int ears, int stride, int kwin,
                                int4* __restrict__ out) {
  const long long total = (long long)dirs * stride;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int2 A = rows[i];
    const int2 B = ears > 1 ? rows[(long long)dirs * stride + i] : make_int2(kwin, 0);
    out[i] = make_int4(A.x, A.y, B.x, B.y);
  }
}

cudaError_t launch_ear_pair_taps(const int2* rows, int dirs, int ears, int stride, int kwin, int4* out,
                                 cudaStream_t st) {
  const long long total = (long long)dirs * stride;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
  k_ear_pair_taps<<<std::max(blocks, 1), 256, 0, st>>>(rows, dirs, ears, stride, kwin, out);
  return cudaGetLastError();
}

cudaError_t launch_pair_taps(const int2* rows, const int* nnz, int n_seg, int seg, int stride, int kwin, int4* out,
                             int4* out_nnz, cudaStream_t st) {
  const long long total = (long long)n_seg * ((seg + 1) / 2) * stride;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
  k_pair_taps<<<std::max(blocks, 1), 256, 0, st>>>(rows, nnz, n_seg, seg, stride, kwin, out, out_nnz);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- launch ----
template <int KWIN, bool STAGE1, int NNZT>
static cudaError_t launch_render_t(const RenderArgs& a, const RenderMaps& m, int sm_count, cudaStream_t st) {
  using C = RenderCfg<KWIN>;
  const SmemLayout L = render_smem_layout(KWIN, STAGE1, a.lf_pad, a.tap_stride);
  auto kern = k_render<KWIN, STAGE1, NNZT>;
  cudaError_t err = ensure_smem(reinterpret_cast<const void*>(kern), L.total);
  if (err != cudaSuccess) return err;
  // TMEM bounds co-residency: at most 512 / COLS CTAs per SM.  Shared memory
  // and registers are sized so the hardware never exceeds that.
  const int per_sm = 512 / C::COLS;
  long long grid = (long long)sm_count * per_sm;
  const long long pairs_total = (a.n_items + 1) / 2;
  if (grid > pairs_total) grid = pairs_total;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, L.total, st>>>(a, m.rows2, m.rows1);
  return cudaGetLastError();
}

template <int KWIN, bool STAGE1>
static cudaError_t dispatch_nnz(const RenderArgs& a, const RenderMaps& m, int sm, cudaStream_t st) {
  if (a.uniform_nnz) {
    switch (a.tap_stride_nnz) {  // == max nnz (all rows equal)
      case 4: return launch_render_t<KWIN, STAGE1, 4>(a, m, sm, st);
      case 8: return launch_render_t<KWIN, STAGE1, 8>(a, m, sm, st);
      case 12: return launch_render_t<KWIN, STAGE1, 12>(a, m, sm, st);
      case 16: return launch_render_t<KWIN, STAGE1, 16>(a, m, sm, st);
      case 24: return launch_render_t<KWIN, STAGE1, 24>(a, m, sm, st);
      case 32: return launch_render_t<KWIN, STAGE1, 32>(a, m, sm, st);
      default: break;
    }
  }
  return launch_render_t<KWIN, STAGE1, 0>(a, m, sm, st);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

cudaError_t make_render_maps(float* out, long long rows, long long out_len, long long out_pitch, RenderMaps* m) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (rows > 1 && (out_pitch * 4) % 16)) return cudaErrorInvalidValue;
  const cuuint64_t dims[2] = {(cuuint64_t)out_len, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(rows > 1 ? out_pitch : ((out_len + 3) / 4 * 4)) * 4};
  const cuuint32_t estr[2] = {1, 1};
  for (int b = 0; b < 2; ++b) {
    const cuuint32_t box[2] = {256, (cuuint32_t)(b == 0 && rows > 1 ? 2 : 1)};
    CUresult r = enc(b == 0 ? &m->rows2 : &m->rows1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

// 3-D map over the rendered rows for the tensor-core kernel: dims {out_len,
// dirs, ears}, box {32 t, 32 directions, 1}; rows past `dirs` (the padding of
// the last 64-direction chunk) and samples past out_len are clipped by TMA.
cudaError_t make_render_mma_map(float* out, int ears, int dirs, long long out_len, long long out_pitch,
                                CUtensorMap* m) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (out_pitch * 4) % 16) return cudaErrorInvalidValue;
  const cuuint64_t dims[3] = {(cuuint64_t)out_len, (cuuint64_t)dirs, (cuuint64_t)ears};
  const cuuint64_t strides[2] = {(cuuint64_t)out_pitch * 4, (cuuint64_t)out_pitch * 4 * dirs};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 2-D map over the mixer's source rows {T, rows} (row pitch `pitch` floats),
// box {kMixTile, 1}: k_mix_mma loads 4 rows per tile::gather4; columns past T
// and rows past `rows` (the K-step padding) are zero-filled by TMA.
cudaError_t make_mix_source_map(const float* y, long long T, long long rows, long long pitch, CUtensorMap* m) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(y) & 15) || (pitch * 4) % 16) return cudaErrorInvalidValue;
  const cuuint64_t dims[2] = {(cuuint64_t)T, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  const cuuint32_t box[2] = {(cuuint32_t)kMixTile, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(y), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int render_kwin_for(int K) {
  if (K <= 113) return 112;
  if (K <= 241) return 240;
  if (K <= 497) return 496;
  return -1;
}

size_t render_smem_bytes(int kwin, bool stage1, int lf_pad, int tap_stride) {
  return (size_t)render_smem_layout(kwin, stage1, lf_pad, tap_stride).total;
}

cudaError_t launch_render(const RenderArgs& a, const RenderMaps& m, int kwin, bool stage1, int sm_count,
                          cudaStream_t st) {
  if (stage1) {
    switch (kwin) {
      case 112: return dispatch_nnz<112, true>(a, m, sm_count, st);
      case 240: return dispatch_nnz<240, true>(a, m, sm_count, st);
      case 496: return dispatch_nnz<496, true>(a, m, sm_count, st);
    }
  } else {
    switch (kwin) {
      case 112: return dispatch_nnz<112, false>(a, m, sm_count, st);
      case 240: return dispatch_nnz<240, false>(a, m, sm_count, st);
      case 496: return dispatch_nnz<496, false>(a, m, sm_count, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace toep
