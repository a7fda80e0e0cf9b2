/*
 * CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, fp64 restatement of the reference toepnmf hot path, used by the
 * parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * *checker*.  The product (paper_1502_03162_b200) never links or calls it.
 *
 * Each routine follows the reference loop structure exactly (same summation
 * order), so results match the reference's compiled backend bit for bit on
 * the same fp64 inputs (pinned against the reference in
 * tests/test_oracle_pin.py and tests/golden/).
 *
 *   orc_conv_dense   <- pkg/src/toepnmf/engine/_kernels.pyx:11-25
 *                       (scatter form out[k+i] += taps[k]*y[i], tap-outer)
 *   orc_conv_sparse  <- pkg/src/toepnmf/engine/_kernels.pyx:28-44
 *                       (out[idx[t]+i] += vals[t]*y[i] over the non-zero taps;
 *                        output length ny+length-1)
 *   orc_render_rows  <- Renderer.render (pkg/src/toepnmf/engine/__init__.py:238-260):
 *                       y*f once per ear (resonance cache), then conv_sparse
 *                       per direction.  Rows are ear-major (row = ear*dirs+d).
 *   orc_mix          <- sum over sources of Renderer.render(y_s, dir(s)) per
 *                       ear, accumulated in fp64 (the mixdown configs have no
 *                       single reference call; this is the composition named
 *                       in SURVEY.md §8c).
 *   orc_mix_window   <- the same restricted to output samples [t0, t0+W):
 *                       every y_s is cropped to [t0-(M-1), t0+W) and rendered
 *                       with the reference loops, which is exact because out[t]
 *                       only depends on y[t-(M-1) .. t].
 * The *_mt drivers spread independent rows / sources over pthreads.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* _kernels.pyx:11-25 */
int64_t orc_conv_dense(const double* y, int64_t ny, const double* taps, int64_t ntaps, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(ny + ntaps - 1));
  int64_t macs = 0;
  for (int64_t k = 0; k < ntaps; ++k) {
    const double tap = taps[k];
    double* o = out + k;
    for (int64_t i = 0; i < ny; ++i) o[i] += tap * y[i];
    macs += ny;
  }
  return macs;
}

/* _kernels.pyx:28-44 */
int64_t orc_conv_sparse(const double* y, int64_t ny, const int64_t* idx, const double* vals, int64_t nnz,
                        int64_t length, double* out) {
  memset(out, 0, sizeof(double) * (size_t)(ny + length - 1));
  int64_t macs = 0;
  for (int64_t t = 0; t < nnz; ++t) {
    const double v = vals[t];
    double* o = out + idx[t];
    for (int64_t i = 0; i < ny; ++i) o[i] += v * y[i];
    macs += ny;
  }
  return macs;
}

/* ------------------------------------------------------------------ rows -- */
typedef struct {
  const double* y;
  int64_t ny;
  const double* f; /* [ears][lf] */
  int64_t lf;
  const int64_t* row_ptr;
  const int64_t* idx;
  const double* vals;
  int64_t K;
  int dirs, ears;
  const int32_t* rows; /* rows to render */
  int nrows;
  double* out; /* [nrows][out_pitch] */
  int64_t out_pitch;
  double* yf; /* [ears][ny+lf-1], computed up front */
  int next;
  pthread_mutex_t mu;
} rows_job;

static void* rows_worker(void* p) {
  rows_job* j = (rows_job*)p;
  const int64_t nyf = j->ny + j->lf - 1;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int i = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (i >= j->nrows) break;
    const int r = j->rows[i];
    const int e = r / j->dirs;
    const int64_t a = j->row_ptr[r], b = j->row_ptr[r + 1];
    orc_conv_sparse(j->yf + (size_t)e * nyf, nyf, j->idx + a, j->vals + a, b - a, j->K,
                    j->out + (size_t)i * j->out_pitch);
  }
  return NULL;
}

/* Renderer.render for a list of rows (engine/__init__.py:238-260). */
int orc_render_rows(const double* y, int64_t ny, const double* f, int64_t lf, int ears, int dirs,
                    const int64_t* row_ptr, const int64_t* idx, const double* vals, int64_t K, const int32_t* rows,
                    int nrows, double* out, int64_t out_pitch, int nthreads) {
  const int64_t nyf = ny + lf - 1;
  rows_job j;
  memset(&j, 0, sizeof(j));
  j.y = y; j.ny = ny; j.f = f; j.lf = lf; j.row_ptr = row_ptr; j.idx = idx; j.vals = vals; j.K = K;
  j.dirs = dirs; j.ears = ears; j.rows = rows; j.nrows = nrows; j.out = out; j.out_pitch = out_pitch;
  j.yf = (double*)malloc(sizeof(double) * (size_t)(nyf * ears));
  if (!j.yf) return -1;
  for (int e = 0; e < ears; ++e) orc_conv_dense(y, ny, f + (size_t)e * lf, lf, j.yf + (size_t)e * nyf);
  pthread_mutex_init(&j.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t th[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, rows_worker, &j);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&j.mu);
  free(j.yf);
  return 0;
}

/* ------------------------------------------------------------------- mix -- */
typedef struct {
  const double* y; /* [S][y_pitch] */
  int64_t T, y_pitch;
  const int32_t* src_dir;
  int S;
  const double* f;
  int64_t lf;
  const int64_t* row_ptr;
  const int64_t* idx;
  const double* vals;
  int64_t K;
  int dirs, ears;
  int64_t t0, W; /* output window */
  double* acc;   /* per-thread [ears][W] */
  int next;
  pthread_mutex_t mu;
} mix_job;

typedef struct {
  mix_job* j;
  double* acc;
} mix_ctx;

static void* mix_worker(void* p) {
  mix_ctx* c = (mix_ctx*)p;
  mix_job* j = c->j;
  const int64_t M = j->lf + j->K - 1;
  /* cropped input [t0-(M-1), t0+W) */
  const int64_t lo = j->t0 - (M - 1);
  const int64_t ncrop = j->W + M - 1;
  double* ycrop = (double*)malloc(sizeof(double) * (size_t)ncrop);
  double* yf = (double*)malloc(sizeof(double) * (size_t)(ncrop + j->lf - 1));
  double* o = (double*)malloc(sizeof(double) * (size_t)(ncrop + M - 1));
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int s = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (s >= j->S) break;
    const double* ys = j->y + (size_t)s * j->y_pitch;
    for (int64_t i = 0; i < ncrop; ++i) {
      const int64_t t = lo + i;
      ycrop[i] = (t >= 0 && t < j->T) ? ys[t] : 0.0;
    }
    for (int e = 0; e < j->ears; ++e) {
      const int r = e * j->dirs + j->src_dir[s];
      const int64_t a = j->row_ptr[r], b = j->row_ptr[r + 1];
      orc_conv_dense(ycrop, ncrop, j->f + (size_t)e * j->lf, j->lf, yf);
      orc_conv_sparse(yf, ncrop + j->lf - 1, j->idx + a, j->vals + a, b - a, j->K, o);
      /* full-conv sample t0+w of the source sits at cropped index (M-1)+w */
      double* acc = c->acc + (size_t)e * j->W;
      for (int64_t w = 0; w < j->W; ++w) acc[w] += o[M - 1 + w];
    }
  }
  free(ycrop);
  free(yf);
  free(o);
  return NULL;
}

/* Mixdown window: out[e][w] = sum_s Renderer_e.render(y_s, dir(s))[t0 + w]. */
int orc_mix_window(const double* y, int64_t T, int64_t y_pitch, const int32_t* src_dir, int S, const double* f,
                   int64_t lf, int ears, int dirs, const int64_t* row_ptr, const int64_t* idx, const double* vals,
                   int64_t K, int64_t t0, int64_t W, double* out, int nthreads) {
  mix_job j;
  memset(&j, 0, sizeof(j));
  j.y = y; j.T = T; j.y_pitch = y_pitch; j.src_dir = src_dir; j.S = S; j.f = f; j.lf = lf;
  j.row_ptr = row_ptr; j.idx = idx; j.vals = vals; j.K = K; j.dirs = dirs; j.ears = ears; j.t0 = t0; j.W = W;
  pthread_mutex_init(&j.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  mix_ctx ctx[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    ctx[t].j = &j;
    ctx[t].acc = (double*)calloc((size_t)ears * W, sizeof(double));
    pthread_create(&th[t], NULL, mix_worker, &ctx[t]);
  }
  memset(out, 0, sizeof(double) * (size_t)(ears * W));
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    for (int64_t i = 0; i < ears * W; ++i) out[i] += ctx[t].acc[i];
    free(ctx[t].acc);
  }
  pthread_mutex_destroy(&j.mu);
  return 0;
}
