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
// Work item = (source group, time tile).  For every source of the group the
// lanes write their 16+KWIN-sample window of y_s into TMEM, then apply the
// source's reflection taps for both ears; the two 16-output accumulators per
// lane persist across the group's sources and are stored once per item.
template <int KWIN>
struct MixSmem {
  static constexpr int COLS = kR + KWIN;
  static constexpr int XH = KWIN + kR;
  static constexpr int kMaxEars = 2;
};

__host__ __device__ inline int mix_smem_floats(int KWIN, int spg, int ears, int tap_stride) {
  const int XH = KWIN + kR;
  int off = ((kW + XH + 31) & ~31);             // source tile
  off += kWarps * 2 * ears * 32 * kR;           // staging (2 slots per ear)
  off += 2 * ears * tap_stride;                 // int2 taps of the current source
  off += ears;                                  // nnz
  (void)spg;
  return off;
}

template <int KWIN, int NNZT>
__global__ void __launch_bounds__(kThreads, 512 / (kR + KWIN)) k_mix(MixArgs a) {
  using C = MixSmem<KWIN>;
  extern __shared__ __align__(128) float smem[];
  __shared__ unsigned s_tbase;
  float* s_x = smem;
  float* s_stage = smem + ((kW + C::XH + 31) & ~31);
  int2* s_taps = reinterpret_cast<int2*>(s_stage + kWarps * 2 * a.ears * 32 * kR);
  int* s_nnz = reinterpret_cast<int*>(s_taps + a.ears * a.tap_stride);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) tmem_alloc<C::COLS>(&s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const unsigned tlane = s_tbase + ((unsigned)(32 * warp) << 16);
  const long long per = (a.n_items + gridDim.x - 1) / gridDim.x;
  const long long it0 = (long long)blockIdx.x * per;
  const long long it1 = min(a.n_items, it0 + per);
  int cur_group = -1;
  int slot = 0;
  float* my_stage = s_stage + warp * 2 * a.ears * 32 * kR;

  for (long long item = it0; item < it1; ++item) {
    const int j = (int)(item % a.n_tiles);
    const int grp = (int)(item / a.n_tiles);
    const long long T0 = (long long)j * kW;
    const int s_begin = grp * a.src_per_group;
    const int ns = min(a.src_per_group, a.S - s_begin);
    (void)cur_group;
    float acc0[16], acc1[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) { acc0[r] = 0.f; acc1[r] = 0.f; }
    for (int s = 0; s < ns; ++s) {
      const float* y = a.y + (long long)(s_begin + s) * a.y_pitch;
      __syncthreads();  // previous source's windows written to TMEM
      const long long xs = T0 - C::XH;
      for (int i = tid; i < kW + C::XH; i += kThreads) {
        const long long t = xs + i;
        s_x[i] = (t >= 0 && t < a.T) ? __ldg(y + t) : 0.f;
      }
      {
        const int dir = a.src_dir[s_begin + s];
        for (int i = tid; i < a.ears * a.tap_stride; i += kThreads) {
          const int e = i / a.tap_stride, k = i % a.tap_stride;
          s_taps[i] = a.taps[((long long)e * a.dirs + dir) * a.tap_stride + k];
        }
        if (tid < a.ears) s_nnz[tid] = a.row_nnz[(long long)tid * a.dirs + dir];
      }
      __syncthreads();
      {
        const int wbase = (C::XH - KWIN) + 16 * tid;
#pragma unroll
        for (int c = 0; c < C::COLS; c += 16) {
          float v[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 t4 = *reinterpret_cast<const float4*>(&s_x[wbase + c + 4 * q]);
            v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
          }
          tmem_st16(tlane + c, v);
        }
        tmem_wait_st();
      }
      for (int e = 0; e < a.ears; ++e) {
        const int2* tp = s_taps + e * a.tap_stride;
        float(&acc)[16] = e ? acc1 : acc0;
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
#pragma unroll
            for (int r = 0; r < 16; ++r) acc[r] = fmaf(v, X[r], acc[r]);
            cur = nxt;
          }
        } else {
          const int nnz = s_nnz[e];
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
      }
    }
    // store the group's partial for this tile
    const long long out_col = T0 + (long long)warp * 32 * kR;
    if (out_col < a.zlen) {
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      for (int e = 0; e < a.ears; ++e) {
        float* st = my_stage + (slot * a.ears + e) * 32 * kR;
        const float(&acc)[16] = e ? acc1 : acc0;
#pragma unroll
        for (int r = 0; r < 16; r += 4)
          *reinterpret_cast<float4*>(&st[lane * 16 + r]) = make_float4(acc[r], acc[r + 1], acc[r + 2], acc[r + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0)
        for (int e = 0; e < a.ears; ++e)
          bulk_store(a.part + ((long long)grp * a.ears + e) * a.part_pitch + out_col,
                     my_stage + (slot * a.ears + e) * 32 * kR, 32 * kR * 4);
      slot ^= 1;
    }
  }
  if (lane == 0) bulk_wait_all();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::COLS>(s_tbase);
}

template <int KWIN, int NNZT>
static cudaError_t launch_mix_t(const MixArgs& a, int sm_count, cudaStream_t st) {
  const int bytes = mix_smem_floats(KWIN, a.src_per_group, a.ears, a.tap_stride) * 4 + 16;
  auto kern = k_mix<KWIN, NNZT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return err;
  const int per_sm = 512 / (kR + KWIN);
  long long grid = (long long)sm_count * per_sm;
  if (grid > a.n_items) grid = a.n_items;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kThreads, bytes, st>>>(a);
  return cudaGetLastError();
}

template <int KWIN>
static cudaError_t mix_nnz(const MixArgs& a, int sm, cudaStream_t st) {
  if (a.uniform_nnz) {
    switch (a.tap_stride) {
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
