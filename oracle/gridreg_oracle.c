/*
 * gridreg_oracle.c -- CPU restatement of the reference DSES hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2502_00115_b200/csrc/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path never links or calls it.
 *
 * It restates, in plain C with IEEE-754 binary64 arithmetic in source order
 * (compile with -ffp-contract=off: the reference's numba kernels contain no
 * FMA), the numba kernels of the reference package
 * `gridreg` (/root/reference/pkg/src/gridreg):
 *
 *   orc_rotation_grid     geometry.py:268-287 (closed-form Rz*Ry*Rx grid) and
 *                         engines.py:120-130 (optional centre pre-multiply)
 *   orc_mode_dense_batch  _kernels.py:109-193 (_mode_dense_one / mode_dense_batch)
 *   orc_point_best        _kernels.py:34-80   (_point_best, metric codes 0..3)
 *   orc_refine_batch      _kernels.py:297-324 (refine_batch)
 *   orc_alignment_error   _kernels.py:83-89   (alignment_error_kernel)
 *
 * Extension (not in the reference): metric code 4 = truncated
 * L2, min(sqrt(min d.d), tau) over the axis-0 window [p0-tau, p0+tau).
 * Parity for code 4 is unpinned by the reference.
 *
 * Parallelism mirrors the reference: rotations are processed in fixed chunks
 * of 16 (_kernels.py:24-26, 181-193) handed out to a pthread pool (numba's
 * prange); every output slot is written by exactly one thread, so results do
 * not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORC_CHUNK 16

enum { ORC_L2 = 0, ORC_L1 = 1, ORC_TRUNC_L1 = 2, ORC_SAT_L0 = 3, ORC_TRUNC_L2 = 4 };

/* ---- minimal pthread parallel-for: workers pull item indices from a shared counter ---- */
typedef struct {
  int64_t next, count;
  pthread_mutex_t mu;
  void (*body)(void* ctx, int64_t item, void* scratch);
  void* (*scratch_new)(void* ctx);
  void* ctx;
  int failed;
} par_job;

static void* par_worker(void* arg) {
  par_job* job = (par_job*)arg;
  void* scratch = job->scratch_new ? job->scratch_new(job->ctx) : NULL;
  if (job->scratch_new && !scratch) {
    pthread_mutex_lock(&job->mu); job->failed = 1; pthread_mutex_unlock(&job->mu);
  }
  for (;;) {
    pthread_mutex_lock(&job->mu);
    const int64_t it = job->failed ? job->count : job->next++;
    pthread_mutex_unlock(&job->mu);
    if (it >= job->count) break;
    job->body(job->ctx, it, scratch);
  }
  free(scratch);
  return NULL;
}

int orc_max_threads(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static int par_for(int64_t count, int nthreads, void (*body)(void*, int64_t, void*),
                   void* (*scratch_new)(void*), void* ctx) {
  par_job job;
  job.next = 0; job.count = count; job.body = body; job.scratch_new = scratch_new;
  job.ctx = ctx; job.failed = 0;
  pthread_mutex_init(&job.mu, NULL);
  if (nthreads <= 0) nthreads = orc_max_threads();
  if (nthreads > count) nthreads = count > 0 ? (int)count : 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  int started = 0;
  for (int t = 1; t < nthreads; ++t)
    if (pthread_create(&th[t], NULL, par_worker, &job) == 0) ++started; else break;
  par_worker(&job);
  for (int t = 1; t <= started; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&job.mu);
  return job.failed ? -1 : 0;
}

/* numpy.searchsorted(a, v, side="left"): first index with a[idx] >= v. */
static int64_t searchsorted_left(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* One grid rotation, geometry.py:272-287.  Angle index a,b,c in [0, 2k];
 * c1,s1 belong to theta (axis X, index a), c2,s2 to phi (b), c3,s3 to xi (c).
 * numpy evaluates `-s3 * c1 + c3 * s2 * s1` as ((-s3)*c1) + ((c3*s2)*s1). */
static void grid_matrix(const double* cth, const double* sth, int64_t a, int64_t b, int64_t c,
                        double* m) {
  const double c1 = cth[a], s1 = sth[a];
  const double c2 = cth[b], s2 = sth[b];
  const double c3 = cth[c], s3 = sth[c];
  m[0] = c3 * c2;
  m[1] = (-s3) * c1 + (c3 * s2) * s1;
  m[2] = s3 * s1 + (c3 * s2) * c1;
  m[3] = s3 * c2;
  m[4] = c3 * c1 + (s3 * s2) * s1;
  m[5] = (-c3) * s1 + (s3 * s2) * c1;
  m[6] = -s2;
  m[7] = c2 * s1;
  m[8] = c2 * c1;
}

/* engines.py:122-126: rots = einsum("ab,lbc->lac", center.R, grid).  The
 * summation order of numpy's einsum is not pinned by the reference; this
 * restatement uses ((C[a0]G[0c] + C[a1]G[1c]) + C[a2]G[2c]). */
static void center_mul(const double* cr, const double* g, double* out) {
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      out[a * 3 + c] = (cr[a * 3 + 0] * g[0 * 3 + c] + cr[a * 3 + 1] * g[1 * 3 + c]) +
                       cr[a * 3 + 2] * g[2 * 3 + c];
}

static void rotation_at(int64_t k, const double* cth, const double* sth, const double* center,
                        int64_t r, double* m) {
  const int64_t n = 2 * k + 1;
  const int64_t a = r / (n * n), b = (r / n) % n, c = r % n;
  if (center) {
    double g[9];
    grid_matrix(cth, sth, a, b, c, g);
    center_mul(center, g, m);
  } else {
    grid_matrix(cth, sth, a, b, c, m);
  }
}

void orc_rotation_grid(int64_t k, const double* cth, const double* sth, const double* center,
                       int64_t r_begin, int64_t r_count, double* out) {
  for (int64_t q = 0; q < r_count; ++q) rotation_at(k, cth, sth, center, r_begin + q, out + 9 * q);
}

/* _kernels.py:109-170, one rotation. counts/last have nbins+1 slots. */
static void mode_dense_one(const double* rot, const double* x, int64_t n, const double* y0,
                           const double* y1, const double* y2, int64_t m, double inv_bin,
                           double bin_size, int64_t lo0, int64_t lo1, int64_t lo2, int64_t d0,
                           int64_t d1, int64_t d2, int32_t* counts, int32_t* last, double* linf,
                           int64_t* best_out, int64_t* lin_out, int64_t* ties_out) {
  const int64_t nbins = d0 * d1 * d2;
  for (int64_t b = 0; b <= nbins; ++b) { counts[b] = 0; last[b] = -1; }
  const double fd0 = (double)d0, fd1 = (double)d1, fd2 = (double)d2;
  const double flo0 = (double)lo0, flo1 = (double)lo1, flo2 = (double)lo2;
  const double dump = (double)nbins;
  for (int64_t i = 0; i < n; ++i) {
    const double xi0 = x[3 * i], xi1 = x[3 * i + 1], xi2 = x[3 * i + 2];
    const double p0 = rot[0] * xi0 + rot[1] * xi1 + rot[2] * xi2;
    const double p1 = rot[3] * xi0 + rot[4] * xi1 + rot[5] * xi2;
    const double p2 = rot[6] * xi0 + rot[7] * xi1 + rot[8] * xi2;
    const double yl = p0 + (flo0 - 1.0) * bin_size;
    const double yh = p0 + (flo0 + fd0) * bin_size;
    const int64_t jlo = searchsorted_left(y0, m, yl);
    const int64_t jhi = searchsorted_left(y0, m, yh);
    for (int64_t j = jlo; j < jhi; ++j) {
      const double q0 = (y0[j] - p0) * inv_bin;
      const double f0 = copysign(floor(fabs(q0) + 0.5), q0) - flo0;
      const double q1 = (y1[j] - p1) * inv_bin;
      const double f1 = copysign(floor(fabs(q1) + 0.5), q1) - flo1;
      const double q2 = (y2[j] - p2) * inv_bin;
      const double f2 = copysign(floor(fabs(q2) + 0.5), q2) - flo2;
      const int ok = (f0 >= 0.0) & (f0 < fd0) & (f1 >= 0.0) & (f1 < fd1) & (f2 >= 0.0) & (f2 < fd2);
      const double v = (f0 * fd1 + f1) * fd2 + f2;
      linf[j] = ok ? v : dump;
    }
    /* _kernels.py:153-158, branch-free: `last[lin] = i` is a no-op when it
     * already holds i, and the dump slot (lin == nbins) is never read back. */
    for (int64_t j = jlo; j < jhi; ++j) {
      const int64_t lin = (int64_t)linf[j];
      const int32_t prev = last[lin];
      last[lin] = (int32_t)i;
      counts[lin] += (prev != (int32_t)i);
    }
  }
  int64_t best = 0, best_lin = -1, ties = 0;
  for (int64_t lin = 0; lin < nbins; ++lin) {
    const int64_t c = counts[lin];
    if (c > best) { best = c; best_lin = lin; ties = 1; }
    else if (c == best && c > 0) { ties += 1; }
  }
  *best_out = best; *lin_out = best_lin; *ties_out = ties;
}

/* _kernels.py:173-193.  Rotations come either from `rots` (nrot x 9) or, when
 * rots == NULL, from the Euler grid (k, cth, sth, center) starting at r_begin. */
typedef struct {
  const double *rots, *cth, *sth, *center, *x, *y0, *y1, *y2;
  int64_t k, r_begin, nrot, n, m, lo0, lo1, lo2, d0, d1, d2;
  double inv_bin, bin_size;
  int64_t *counts_out, *lins_out, *ties_out;
} mode_ctx;

typedef struct { int32_t* counts; int32_t* last; double* linf; } mode_scratch;

static void* mode_scratch_new(void* vctx) {
  const mode_ctx* c = (const mode_ctx*)vctx;
  const int64_t nbins = c->d0 * c->d1 * c->d2;
  /* one allocation so the pool can free() it with a single call:
   * [header | pad to 32 B | linf f64[m] | counts i32[nbins+1] | last i32[nbins+1]] */
  const size_t nb = (size_t)(nbins + 1), nm = (size_t)(c->m > 0 ? c->m : 1);
  const size_t head = 32;
  char* blob = (char*)malloc(head + sizeof(double) * nm + 2 * sizeof(int32_t) * nb);
  if (!blob) return NULL;
  mode_scratch* s = (mode_scratch*)blob;
  s->linf = (double*)(blob + head);
  s->counts = (int32_t*)(s->linf + nm);
  s->last = s->counts + nb;
  return s;
}

static void mode_chunk(void* vctx, int64_t chunk, void* vs) {
  const mode_ctx* c = (const mode_ctx*)vctx;
  mode_scratch* s = (mode_scratch*)vs;
  const int64_t hi = (chunk + 1) * ORC_CHUNK < c->nrot ? (chunk + 1) * ORC_CHUNK : c->nrot;
  for (int64_t r = chunk * ORC_CHUNK; r < hi; ++r) {
    double rbuf[9];
    const double* rot;
    if (c->rots) rot = c->rots + 9 * r;
    else { rotation_at(c->k, c->cth, c->sth, c->center, c->r_begin + r, rbuf); rot = rbuf; }
    mode_dense_one(rot, c->x, c->n, c->y0, c->y1, c->y2, c->m, c->inv_bin, c->bin_size, c->lo0,
                   c->lo1, c->lo2, c->d0, c->d1, c->d2, s->counts, s->last, s->linf,
                   &c->counts_out[r], &c->lins_out[r], &c->ties_out[r]);
  }
}

/* Returns 0, or -1 when scratch allocation fails. */
int orc_mode_dense_batch(const double* rots, int64_t k, const double* cth, const double* sth,
                         const double* center, int64_t r_begin, int64_t nrot, const double* x,
                         int64_t n, const double* y0, const double* y1, const double* y2, int64_t m,
                         double inv_bin, double bin_size, int64_t lo0, int64_t lo1, int64_t lo2,
                         int64_t d0, int64_t d1, int64_t d2, int64_t* counts_out, int64_t* lins_out,
                         int64_t* ties_out, int nthreads) {
  mode_ctx c = {rots, cth, sth, center, x, y0, y1, y2, k, r_begin, nrot, n, m, lo0, lo1, lo2,
                d0, d1, d2, inv_bin, bin_size, counts_out, lins_out, ties_out};
  const int64_t nchunks = (nrot + ORC_CHUNK - 1) / ORC_CHUNK;
  return par_for(nchunks, nthreads, mode_chunk, mode_scratch_new, &c);
}

/* _kernels.py:34-80 (codes 0..3) plus the code-4 extension. */
static double point_best(double p0, double p1, double p2, const double* y0, const double* y1,
                         const double* y2, int64_t m, int code, double param) {
  if (code == ORC_TRUNC_L1) {
    const int64_t jlo = searchsorted_left(y0, m, p0 - param);
    const int64_t jhi = searchsorted_left(y0, m, p0 + param);
    double best = param;
    for (int64_t j = jlo; j < jhi; ++j) {
      const double v = fabs(y0[j] - p0) + fabs(y1[j] - p1) + fabs(y2[j] - p2);
      if (v < best) { best = v; if (best == 0.0) break; }
    }
    return best;
  }
  if (code == ORC_SAT_L0) {
    const double half = 0.5 * param;
    const int64_t jlo = searchsorted_left(y0, m, p0 - half);
    const int64_t jhi = searchsorted_left(y0, m, p0 + half);
    for (int64_t j = jlo; j < jhi; ++j)
      if (fabs(y0[j] - p0) < half && fabs(y1[j] - p1) < half && fabs(y2[j] - p2) < half) return 0.0;
    return 1.0;
  }
  if (code == ORC_L1) {
    double best = INFINITY;
    for (int64_t j = 0; j < m; ++j) {
      const double v = fabs(y0[j] - p0) + fabs(y1[j] - p1) + fabs(y2[j] - p2);
      if (v < best) best = v;
    }
    return best;
  }
  if (code == ORC_TRUNC_L2) { /* extension: parity unpinned by the reference */
    const int64_t jlo = searchsorted_left(y0, m, p0 - param);
    const int64_t jhi = searchsorted_left(y0, m, p0 + param);
    const double cap = param * param;
    double best = cap;
    for (int64_t j = jlo; j < jhi; ++j) {
      const double d0 = y0[j] - p0, d1 = y1[j] - p1, d2 = y2[j] - p2;
      const double v = d0 * d0 + d1 * d1 + d2 * d2;
      if (v < best) best = v;
    }
    return best < cap ? sqrt(best) : param;
  }
  double best = INFINITY;
  for (int64_t j = 0; j < m; ++j) {
    const double d0 = y0[j] - p0, d1 = y1[j] - p1, d2 = y2[j] - p2;
    const double v = d0 * d0 + d1 * d1 + d2 * d2;
    if (v < best) best = v;
  }
  return sqrt(best);
}

double orc_point_best(double p0, double p1, double p2, const double* y0, const double* y1,
                      const double* y2, int64_t m, int code, double param) {
  return point_best(p0, p1, p2, y0, y1, y2, m, code, param);
}

/* _kernels.py:83-89: serial fixed-order sum over already-transformed points. */
double orc_alignment_error(const double* p, int64_t n, const double* y0, const double* y1,
                           const double* y2, int64_t m, int code, double param) {
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i)
    total += point_best(p[3 * i], p[3 * i + 1], p[3 * i + 2], y0, y1, y2, m, code, param);
  return total;
}

/* _kernels.py:297-324: one output slot per candidate pose. */
typedef struct {
  const double *rots, *ts, *x, *y0, *y1, *y2;
  int64_t n, m; int code; double param; double* out;
} refine_ctx;

static void refine_one(void* vctx, int64_t c, void* unused) {
  (void)unused;
  const refine_ctx* k = (const refine_ctx*)vctx;
  const double* r = k->rots + 9 * c;
  const double t0 = k->ts[3 * c], t1 = k->ts[3 * c + 1], t2 = k->ts[3 * c + 2];
  double total = 0.0;
  for (int64_t i = 0; i < k->n; ++i) {
    const double xi0 = k->x[3 * i], xi1 = k->x[3 * i + 1], xi2 = k->x[3 * i + 2];
    const double p0 = r[0] * xi0 + r[1] * xi1 + r[2] * xi2 + t0;
    const double p1 = r[3] * xi0 + r[4] * xi1 + r[5] * xi2 + t1;
    const double p2 = r[6] * xi0 + r[7] * xi1 + r[8] * xi2 + t2;
    total += point_best(p0, p1, p2, k->y0, k->y1, k->y2, k->m, k->code, k->param);
  }
  k->out[c] = total;
}

void orc_refine_batch(const double* rots, const double* ts, int64_t ncand, const double* x,
                      int64_t n, const double* y0, const double* y1, const double* y2, int64_t m,
                      int code, double param, double* out, int nthreads) {
  refine_ctx k = {rots, ts, x, y0, y1, y2, n, m, code, param, out};
  par_for(ncand, nthreads, refine_one, NULL, &k);
}
