// Internal launcher interface between the C ABI (capi.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <mutex>
#include <unordered_map>

namespace toep {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last granted on this device (a per-launch call costs
// microseconds of host time on the latency paths).
inline cudaError_t ensure_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::unordered_map<long long, int> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const long long key = (long long)(reinterpret_cast<uintptr_t>(func) ^ ((uintptr_t)dev << 48));
  std::lock_guard<std::mutex> lk(mu);
  int& cur = granted[key];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

constexpr int kR = 16;             // outputs per lane (one TMEM x16 load per tap)
constexpr int kWarps = 4;          // warps per CTA: one per TMEM lane quarter
constexpr int kThreads = 32 * kWarps;
constexpr int kW = kThreads * kR;  // outputs per CTA tile (2048)

// Tap tables are row-major "ELL" arrays of int2 {col, value-bits} with
// col = KWIN - offset (the TMEM window column where the tap's 16-sample
// slice starts) and a per-row count in row_nnz.  Rows are ear-major:
// row = ear * dirs + direction.
struct RenderArgs {
  const float* x;        // stage1: source signal y[nx]; else y*f per ear at x + ear*x_pitch
  long long nx;          // input length
  long long x_pitch;     // per-ear input stride (stage-2-only mode)
  const float* f;        // [ears][lf_pad] resonance taps, zero padded (stage1)
  int lf_pad;            // multiple of 16
  const int4* pairs;     // [ears][pairs_per_ear][tap_stride] {colA, vA, colB, vB} (k_pair_taps)
  const int4* pair_nnz;  // [ears][pairs_per_ear] {nnzA, nnzB, 0, 0}
  int pairs_per_ear;     // ceil(dirs / 2)
  int tap_stride;        // entries per row (>= max nnz, even)
  int uniform_nnz;       // 1 if every row holds exactly tap_stride_nnz taps
  int tap_stride_nnz;
  int dirs;              // directions per ear
  int ears;
  int n_tiles;           // ceil(out_len / 2048)
  long long n_items;     // work units: ears * dirs * n_tiles
  float* out;            // row r at out + r * out_pitch
  long long out_pitch;   // floats, multiple of 4, >= n_tiles*2048 rounded down to 512 granularity
  long long out_len;
  int* nonfinite;        // set to 1 when a non-finite input sample is read (may be null)
};

// Tensor-core renderer (render_mma.cu): stage 2 as a split-fp16 GEMM per
// (ear, 128-output tile, 128-direction chunk) unit.
struct RenderMmaArgs {
  const float* x;        // source y[nx]
  long long nx;
  const float* f;        // [ears][lf_pad] resonance taps, zero padded
  int lf_pad;
  const void* g;         // [ears][nchunks][hi, lo][canonical chunk x kpad] fp16 (build_render_mma_tables)
  const int* gexp;       // [ears][nchunks][128 + 1] G row exponents + "wide chunk" flag (build_render_mma_tables)
  int kpad;              // round_up(K, 16)
  int nchunks;           // ceil(dirs / render_mma_chunk())
  int dirs, ears;
  int n_titems;          // ceil(out_len / 128)
  int t_begin, t_end;    // this launch's 128-output tiles of every ear (set by launch_render_mma)
  float* out;            // row (e * dirs + d) at out + row * out_pitch
  long long out_pitch;
  long long out_len;
  int* nonfinite;
};
bool render_mma_supported(int K, int lf_pad);
int render_mma_kpad(int K);
int render_mma_chunk();  // directions per G chunk (MMA N)
size_t render_mma_gbytes(int ears, int dirs, int K);
size_t render_mma_gexp_ints(int ears, int dirs);
cudaError_t build_render_mma_tables(const int2* raw, const int* nnz, int dirs, int ears, int stride, int K,
                                    void* g, int* gexp, cudaStream_t st);
cudaError_t make_render_mma_map(float* out, int ears, int dirs, long long out_len, long long out_pitch,
                                CUtensorMap* m);
// side stream + fork/join events of one renderer (the concurrent fill launch)
struct MmaFillStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t launch_render_mma(const RenderMmaArgs& a, const CUtensorMap& map, const MmaFillStreams& fs, int sm_count,
                              cudaStream_t st);
int render_mma_launches(int n_titems, int kpad, int lf_pad, int sm_count);

// FFT (fft.cu): radix-2, power-of-two n; complex buffers interleaved.
cudaError_t launch_fft_c128(const double* in, double* out, long long n, bool inverse, cudaStream_t st);
cudaError_t launch_fft_c64(const float* in, float* out, long long n, long long batch, bool inverse, cudaStream_t st);
cudaError_t launch_fft_conv(const float* y, long long ny, const float* spectrum, long long n, long long ntaps,
                            float* out, float* scratch, cudaStream_t st);
cudaError_t launch_fft_spectrum(const float* taps, long long ntaps, long long n, float* spectrum, float* tmp,
                                cudaStream_t st);
long long fft_conv_scratch_bytes(long long ny, long long n, long long ntaps);
bool fft_needs_distinct(long long n, bool dbl);

// TMA tensor maps over the output rows ([rows][out_len], row stride out_pitch):
// box {256, 2} for direction pairs and {256, 1} for a trailing odd direction.
struct RenderMaps {
  alignas(64) CUtensorMap rows2;
  alignas(64) CUtensorMap rows1;
};

int render_kwin_for(int K);
size_t render_smem_bytes(int kwin, bool stage1, int lf_pad, int tap_stride);
cudaError_t launch_pair_taps(const int2* rows, const int* nnz, int n_seg, int seg, int stride, int kwin, int4* out,
                             int4* out_nnz, cudaStream_t st);
cudaError_t make_render_maps(float* out, long long rows, long long out_len, long long out_pitch, RenderMaps* m);
cudaError_t launch_render(const RenderArgs& a, const RenderMaps& m, int kwin, bool stage1, int sm_count,
                          cudaStream_t st);

// Dense FIR, one filter per channel: out[c][t] = sum_j h[c][j] x[c][t-j], t < out_len.
struct FirArgs {
  const float* x;
  long long nx;
  long long x_pitch;
  const float* h;        // [channels][h_pitch]; taps past nh read as zero
  int nh_pad;            // nh rounded up to 16 (the loop structure)
  int nh;                // taps actually stored per channel
  int h_pitch;
  float* out;
  long long out_len;
  long long out_pitch;
  int channels;
};
cudaError_t launch_fir(const FirArgs& a, cudaStream_t st);

// Generic sparse convolution for long reflection filters (K > 497): banded
// shared-memory gather.  Same tap encoding but col = raw offset.
struct SparseGenericArgs {
  const float* x;
  long long nx;
  long long x_pitch;     // input stride between row groups (0 = shared input)
  int rows_per_x;        // consecutive rows sharing one input (>= 1)
  const int2* taps;      // raw offsets
  const int* row_nnz;
  int tap_stride;
  int rows;
  float* out;
  long long out_len;
  long long out_pitch;
};
cudaError_t launch_sparse_generic(const SparseGenericArgs& a, cudaStream_t st);

// Source -> per-ear partial mix, reflection filters first (g-first order):
//   part[grp][e][t] = sum_{s in grp} sum_k v_{e,d(s),k} * y_s[t - o_{e,d(s),k}]
// Bucketed mix (one pass over the sources): buckets are the sets of sources
// sharing a direction; item = (bucket group, 2048-sample tile).
constexpr int kMixMaxBuckets = 512;    // buckets per group
constexpr int kMixGroupSrcCap = 1024;  // sources per bucket group (host splits larger buckets)
struct MixArgs {
  const float* y;        // sources, row s at y + s * y_pitch, length T
  long long T;
  long long y_pitch;
  const int* bsrc;       // sources ordered by bucket
  const int* bptr;       // [buckets + 1]
  const int* bdir;       // [buckets] direction of each bucket
  int buckets;
  int buckets_per_group;
  int group_srcs;        // shared-memory source-table capacity (>= every group's source count)
  int groups;
  int n_tiles;           // ceil(zlen / 2048)
  long long n_items;     // groups * n_tiles
  const int2* taps;      // ear-major [ears * dirs][tap_stride], col = KWIN - o
  const int4* etaps;     // [dirs][tap_stride] {col_e0, v_e0, col_e1, v_e1} (k_ear_pair_taps)
  const int* row_nnz;
  int tap_stride;
  int dirs;
  int ears;
  float* part;           // [groups][ears][part_pitch]
  unsigned long long* work;  // item counter for dynamic scheduling (zeroed before the launch), or null
  long long part_pitch;
  long long zlen;        // T + K - 1
  int* nonfinite;        // set to 1 when a non-finite source sample is read (may be null)
};
cudaError_t launch_mix(const MixArgs& a, int kwin, int nnz_uniform, int sm_count, cudaStream_t st);
cudaError_t launch_ear_pair_taps(const int2* rows, int dirs, int ears, int stride, int kwin, int4* out,
                                 cudaStream_t st);

// Tensor-core mixdown (mix_mma.cu): W[t][(e,o)] = sum_d Y_d[t] G[d][(e,o)] on
// tcgen05 (M = 128 time rows, K = 16 direction rows per step, N = ears x KP),
// then z_e[t] = sum_o W[t-o][(e,o)].  The host plans K-steps of up to 16 rows
// (a row = up to kMixRowSrcs sources of one direction; one row size per K-step).
constexpr int kMixTile = 256;     // samples per tile (two 128-row blocks of the MMA)
constexpr int kMixRowSrcs = 4;    // sources per direction row
constexpr int kMixKsSrcs = 64;    // sources per K-step
struct MixMmaArgs {
  const float* y;        // sources, row i at y + i * y_pitch (16-byte aligned rows), length T
  long long T;
  long long y_pitch;
  const unsigned short* src;  // source rows in K-step order, each K-step padded to a multiple of 4 (tensor-map rows)
  const int2* ks;        // [KS] {first entry in src (multiple of 4), padded count}
  const int* rows;       // [KS][16] row r: offset | count << 6 | (gamma_d + 128) << 9
  const float* rowf;     // [KS][16] main-pass multiplier 2^(sexp - gamma_d) of row r
  const unsigned char* g;  // [KS][hi, lo][canonical N x 16] fp16 of g * 2^gamma_d
  int KS;
  int nsrc4;             // entries of src (all K-steps, padded)
  int ring;              // 512-byte source slots in shared memory (mix_mma_ring)
  int N;                 // MMA N (multiple of 16, <= 208)
  int KP;                // columns per ear (K rounded up to 8)
  int K;                 // reflection length
  int ears;
  int n_tiles;           // ceil(T / kMixTile)
  int sexp;              // launch scale 2^sexp of the A operand
  float* z;              // [ears][z_pitch], z_len = T + K - 1
  long long z_pitch;
  long long zlen;
  float* ovh;            // [n_tiles][ears][ovh_pitch] overlap-add tails
  int ovh_pitch;
  float* tile_max;       // [n_tiles] max |Y_d 2^-gamma_d| per tile
  const int* bad_list;   // fixup pass: tiles to re-render (null: every tile)
  const int* bad_count;
  int* nonfinite;
  int* scan_list;        // main pass: where the last CTA lists the fixup tiles (null: no scan)
  int* scan_count;
  unsigned* scan_done;   // CTA arrival counter (zero between calls)
};
// main pass (its last CTA lists the tiles for the fixup pass), fixup pass,
// finish (overhang carry + z finite check): 3 launches; bad_count[1] is the
// main pass's arrival counter and must be zero before the first call
// tm: 2-D tensor map over the sources {T, rows}, box {kMixTile, 1} (tile::gather4 loads)
cudaError_t launch_mix_mma(const MixMmaArgs& a, const CUtensorMap& tm, int* bad_list, int* bad_count, int sm_count,
                           cudaStream_t st);
cudaError_t make_mix_source_map(const float* y, long long T, long long rows, long long pitch, CUtensorMap* m);
// shared-memory source-ring slots left next to the K-step tables; 0 = the tables do not fit
int mix_mma_ring(int N, int ears, int K, int nsrc4, int KS);

// z[e][t] = sum_g part[g][e][t]  (fixed order, fp32)
cudaError_t launch_mix_reduce(const float* part, int groups, int ears, long long part_pitch, long long zlen,
                              float* z, long long z_pitch, cudaStream_t st);

// Streaming block step (g-first, carried history).
#ifndef TOEP_STREAM_GROUP
#define TOEP_STREAM_GROUP 16
#endif
constexpr int kStreamGroup = TOEP_STREAM_GROUP;  // CTAs per first-level reduction group of k_stream_step
constexpr int kStreamCL = 8;  // CTAs per cluster of k_stream_cl (the default streaming kernel)
// CTAs of a streaming step for S sources, spc per CTA (a multiple of kStreamCL for k_stream_cl)
int stream_ctas(int S, int spc, bool cluster);
bool stream_cluster_enabled();
struct StreamArgs {
  const float* block;    // new samples, source s at block + s * block_pitch
  long long block_pitch;
  int B;
  float* yhist;          // [S][H] last H samples of every source (H >= K-1, multiple of 4)
  int H;
  int S;
  const int2* src_taps;  // [S][ears][tap_stride] raw taps (col = o) of each source's direction
  const int* src_nnz;    // [S][ears]
  int tap_stride;
  int ears;
  int src_per_cta;
  float* part;           // [ctas][ears][B] per-CTA z partials
  float* gpart;          // [groups][ears][B] f * (group z)
  float* zhist;          // [groups][ears][zh] last zh samples of each group's z
  int zh;                // z history length (lf_pad >= Lf - 1)
  const float* f;        // [ears][lf_pad]
  int lf_pad;
  float* out;            // ear e at out + e * out_pitch, B samples
  long long out_pitch;
  int ctas;
  unsigned int* ticket;  // [groups + 1] zero-initialised counters owned by the stream state
  int* nonfinite;        // set to 1 when a non-finite input sample is read (may be null)
  int cluster;           // 1: k_stream_cl (clusters of kStreamCL CTAs), 0: k_stream_step
};
cudaError_t launch_stream_gather_taps(const int2* raw, const int* nnz, const int* src_dir, int S, int ears, int dirs,
                                      int stride, int2* out, int* out_nnz, cudaStream_t st);
cudaError_t launch_stream_step(const StreamArgs& a, cudaStream_t st);

}  // namespace toep
