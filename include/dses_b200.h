/*
 * dses_b200.h -- C ABI of the B200-native DSES (Direct Semi-Exhaustive Search)
 * registration hot path.  No torch or CUDA types appear in these signatures:
 * pointers are plain host pointers unless a name ends in `_dev`, sizes are
 * int64, the CUDA stream is passed as `void*` (a cudaStream_t; NULL = the
 * legacy default stream).
 *
 * Reference interfaces replaced (reference = gridreg 0.1.0 under
 * /root/reference/pkg/src/gridreg):
 *
 *   dses_mode_dense_batch  <- _kernels.mode_dense_batch   (_kernels.py:173-193)
 *                             (and mode_sparse_batch, _kernels.py:277-294:
 *                             same outputs for any lattice size)
 *   dses_refine_batch      <- _kernels.refine_batch       (_kernels.py:297-324); with one
 *                             pose it is alignment_error_kernel (_kernels.py:83-89)
 *                             after RigidTransform.apply (metrics.py:133-140)
 *   dses_exhaustive        <- engines.exhaustive_search   (engines.py:156-193)
 *   dses_plan_* + dses_search / dses_stage_*
 *                          <- engines.dses                (engines.py:229-301),
 *                             split into the stages a multi-GPU caller needs
 *                             between its collectives.
 *
 * Every function returns 0 on success or a negative DSES_E* code; the text of
 * the last error on the calling thread is available from dses_last_error().
 * Validation that the reference performs in Python (shapes, finiteness, grid
 * extent, caps) stays in the Python host layer, which raises the reference's
 * exception types; this layer only rejects what would be undefined behaviour.
 */
#ifndef DSES_B200_H
#define DSES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSES_OK 0
#define DSES_E_INVALID -1   /* bad argument (would be InvalidInputError upstream) */
#define DSES_E_CUDA -2      /* CUDA runtime / launch failure */
#define DSES_E_NOMEM -3     /* device or host allocation failed */
#define DSES_E_NODEVICE -4  /* no CUDA device / the sm_100a image cannot run here */
#define DSES_E_LIMIT -5     /* input beyond a documented size limit of this implementation
                               (SearchSpaceTooLargeError upstream) */

/* Metric codes follow _kernels.py:15-16 (METRIC_*), plus code 4 (extension). */
#define DSES_METRIC_L2 0
#define DSES_METRIC_L1 1
#define DSES_METRIC_TRUNC_L1 2
#define DSES_METRIC_SAT_L0 3
#define DSES_METRIC_TRUNC_L2 4 /* extension; not in the reference */

typedef struct dses_plan dses_plan; /* opaque: one (source, reference, lattice) problem on one GPU */

/* Rotation source: the lexicographic Euler grid of geometry.py:253-290 given by
 * its per-axis cos/sin tables (index a in [0, 2k] <-> angle (a - k) * step,
 * computed by the caller exactly as geometry.py:272-275 does), optionally
 * left-multiplied by a centre rotation (engines.py:122-126). */
typedef struct {
  int64_t k;              /* half width; (2k+1)^3 rotations */
  const double* cos_tab;  /* host, 2k+1 values */
  const double* sin_tab;  /* host, 2k+1 values */
  const double* center;   /* host, 9 values row-major, or NULL */
} dses_grid;

/* Outcome of one search (or one rank's share of it). */
typedef struct {
  int64_t candidates_evaluated; /* rotations with an in-window vote (engines.py:254,293) */
  int64_t candidates_refined;   /* n_score (engines.py:270,294); 0 on the sat_l0 shortcut */
  int64_t mstar;                /* best vote count M* */
  int64_t winner_row;           /* flat rotation index of the winner (lexicographic grid order) */
  int64_t winner_lin;           /* flat translation-bin index of the winner's mode */
  int64_t winner_count;         /* its vote count */
  double best_error;            /* metric error of the winner (refine_batch op order) */
  int64_t best_inliers;         /* count_inliers at trans_bin (metrics.py:143-150) */
  int64_t rescored;             /* candidates re-scored in exact fp64 */
  /* kernel statistics */
  int64_t pairs_evaluated;      /* (rotation, i, j) pairs the vote kernel tested */
  int64_t votes;                /* deduplicated in-window votes (histogram increments) */
  int64_t rechecks;             /* pairs re-binned in fp64 (fixed-point guard band) */
  double ms_vote, ms_select, ms_score, ms_total; /* device time per stage (CUDA events) */
  double ms_vote_kernel;        /* the vote kernel alone (events around its launch) */
  int64_t launches;             /* kernels this plan launched since its counters were reset */
  int64_t h2d_bytes, d2h_bytes; /* host<->device bytes copied for this plan since the reset */
} dses_result;

const char* dses_last_error(void);
int dses_device_count(int* out);
const char* dses_build_info(void);
/* A non-blocking CUDA stream on `device` (an opaque cudaStream_t for the
 * `stream` arguments); destroy synchronises it first.  Two of them let
 * consecutive registrations overlap at their boundaries (engines.dses_batch). */
int dses_stream_create(int device, void** stream);
int dses_stream_destroy(void* stream);

/* ---- plan lifecycle ----------------------------------------------------- */
/* x: source (n,3) row-major f64; y: reference (m,3).  bin_size = trans_bin;
 * ilo/dims: inclusive lower bin index and bin counts of the translation
 * window (engines.py:248-250).  Copies x, y to `device`. */
int dses_plan_create(int device, const double* x, int64_t n, const double* y, int64_t m,
                     double bin_size, const int64_t ilo[3], const int64_t dims[3],
                     dses_plan** out);
int dses_plan_destroy(dses_plan* plan);
/* Fixed-point fraction bits chosen for the vote kernel (0 = exact fp64 mode). */
int dses_plan_info(const dses_plan* plan, int64_t* frac_bits, int64_t* x_tiles, int64_t* y_tiles,
                   int64_t* near_pairs);
/* Testing hook: run the vote kernel on at most `ctas` persistent CTAs
 * (0 = the default, one wave of resident CTAs).  Results do not depend on it
 * (tests/test_gpu_api.py checks 1, 7 and 148 CTAs against the default). */
int dses_plan_set_vote_grid(dses_plan* plan, int64_t ctas);
/* Rotation blocks: boxes of shape[0] x shape[1] x shape[2]
 * neighbouring grid rotations (along the three Euler-index axes, at most 32
 * rotations) share one candidate-pair list; 0,0,0 = the per-rotation vote
 * kernel.  Default: 1,3,3 when few reference points of a group fall in a
 * source point's window (estimated lane use of the per-rotation kernel below
 * 0.2), else 0,0,0 (environment DSES_BLOCK_SHAPE="a,b,c"
 * overrides); plans with n * m_pad >= 2^28 always take the per-rotation
 * kernel.  list_cap: 16-byte list entries per CTA (0 = default 2^17, 2 MiB;
 * blocks whose list overflows are re-run by the per-rotation kernel).
 * Results do not depend on either. */
int dses_plan_set_blocks(dses_plan* plan, const int64_t shape[3], int64_t list_cap);
/* The block shape this plan's grid searches use (0,0,0: per-rotation kernel). */
int dses_plan_blocks(const dses_plan* plan, int64_t shape[3]);

/* ---- the reference kernel seams ------------------------------------------ */
/* Per-rotation histogram mode (count, flat bin, tied bins) for `nrot`
 * rotations given explicitly (rots: host (nrot,3,3) f64) -- _kernels.py:173. */
int dses_mode_batch(dses_plan* plan, const double* rots, int64_t nrot, int64_t* counts,
                    int64_t* lins, int64_t* ties, void* stream);
/* Same for rotations [r_begin, r_begin + nrot) of an Euler grid. */
int dses_mode_grid(dses_plan* plan, const dses_grid* grid, int64_t r_begin, int64_t nrot,
                   int64_t* counts, int64_t* lins, int64_t* ties, void* stream);
/* Full translation vote map of ONE rotation (rot: host (3,3) f64) over the
 * plan's lattice -- mode_search.translation_histogram (mode_search.py:205-235):
 * bins in ascending flat order with their counts (distinct source points per
 * bin when `dedup`, raw pair votes otherwise).  Pair bins use the vote
 * kernel's binary64 operation order (_kernels.py:244-253).  *nbins = number of
 * non-empty bins (DSES_E_INVALID if > cap; cap = n*m always suffices),
 * *npairs (optional) = pairs inside the lattice. */
int dses_translation_histogram(dses_plan* plan, const double* rot, int dedup, int64_t* lins,
                               int64_t* counts, int64_t cap, int64_t* nbins, int64_t* npairs,
                               void* stream);
/* Exact fp64 alignment error of `ncand` poses (rots (c,3,3), ts (c,3)) in
 * refine_batch's operation order -- _kernels.py:297-324. */
int dses_refine_batch(dses_plan* plan, const double* rots, const double* ts, int64_t ncand,
                      int metric_code, double param, double* out, void* stream);
/* Stand-alone mode_dense_batch with the reference's exact signature meaning
 * (creates and destroys a transient plan on `device`). */
int dses_mode_dense_batch(int device, const double* rots, int64_t nrot, const double* x, int64_t n,
                          const double* y, int64_t m, double bin_size, const int64_t ilo[3],
                          const int64_t dims[3], int64_t* counts, int64_t* lins, int64_t* ties);

/* ---- the full search ---------------------------------------------------- */
/* engines.dses phases 1-3 on one GPU over rotations [r_begin, r_begin+r_count)
 * of `grid` (r_count < 0: the whole grid). */
int dses_search(dses_plan* plan, const dses_grid* grid, int64_t r_begin, int64_t r_count, double q,
                int metric_code, double metric_param, int skip_refine, dses_result* out,
                void* stream);
/* Allocate every device buffer a search over `r_count` rotations uses (also
 * done at the top of each search; calling it at plan construction keeps
 * memory-pool growth off the search's timeline). */
int dses_plan_reserve(dses_plan* plan, int64_t r_count);
/* dses_search split in two: _async enqueues the whole search on `stream` and
 * returns (grid's host tables must stay valid until _wait); _wait blocks on
 * it and fills `out`.  Lets a caller queue registration k+1 before reading
 * the result of k (engines.dses_batch).  One search in flight per plan. */
int dses_search_async(dses_plan* plan, const dses_grid* grid, int64_t r_begin, int64_t r_count,
                      double q, int metric_code, double param, int skip_refine, void* stream);
int dses_search_wait(dses_plan* plan, dses_result* out);

/* engines.exhaustive_search (engines.py:156-193, _kernels.exhaustive_batch
 * _kernels.py:327-381): the metric at every pose of the 6-D grid, rotations
 * of `grid` x translations t_center + (-k..k) * trans_bin per axis; winner =
 * minimum error, ties to the smallest (rotation, translation) enumeration
 * index.  winner_row / winner_lin = rotation / translation flat index,
 * best_error = its binary64 error (refine_batch operation order). */
int dses_exhaustive(dses_plan* plan, const dses_grid* grid, int64_t k_trans,
                    const double t_center[3], int metric_code, double metric_param,
                    dses_result* out, void* stream);

/* ---- stages for a sharded (multi-GPU) search ----------------------------- */
/* Stage 1: vote over this rank's rotation slice; returns local M* and the
 * local count of rotations with an in-window vote. */
int dses_stage_vote(dses_plan* plan, const dses_grid* grid, int64_t r_begin, int64_t r_count,
                    int64_t* mstar_local, int64_t* valid_local, void* stream);
/* Stage 2 (shortcut path): smallest local row whose count equals the global
 * M* (INT64_MAX when none). */
int dses_stage_argmax(dses_plan* plan, int64_t mstar_global, int64_t* row_local, void* stream);
/* Stage 2: keep local rows with count >= q*M*_global - 1e-9 (engines.py:196-201),
 * screen them in fp32; returns the local kept count and the local fp32 minimum
 * (+inf when none) and the screen tolerance (absolute). */
int dses_stage_screen(dses_plan* plan, double q, int64_t mstar_global, int metric_code,
                      double metric_param, int64_t* kept_local, double* min32_local,
                      double* tol, void* stream);
/* Stage 3: exact fp64 re-score of local kept rows with screen error <=
 * threshold; returns the local (error, row) minimum (error +inf when none). */
int dses_stage_rescore(dses_plan* plan, double threshold, int metric_code, double metric_param,
                       double* err_local, int64_t* row_local, int64_t* rescored, void* stream);
/* Translation-bin index (flat) of a local row's mode. */
int dses_stage_row_info(dses_plan* plan, int64_t row, int64_t* lin, int64_t* count, void* stream);
/* Exact fp64 error of one pose (grid row + translation bin) under a metric --
 * metrics.alignment_error with refine_batch's operation order. */
int dses_pose_error(dses_plan* plan, const dses_grid* grid, int64_t row, int64_t lin,
                    int metric_code, double metric_param, double* err, void* stream);
/* Kernel statistics accumulated since the last call (pairs, votes, rechecks). */
/* ---- device-resident sharded search --------------------
 * engines.dses with the rotation grid split over ranks, exchange values kept
 * in DEVICE memory: `xchg` is an int64[7] device buffer of the caller that it
 * reduces with NCCL between the calls (all on `stream`, no host round trip):
 *   dses_shard_vote    vote over the rank's slice; x[0] = local M*, x[3] =
 *                      rotations with a vote               -> all_reduce x[0] MAX
 *   dses_shard_select  cutoff from the GLOBAL M* in x[0], fp32 screen, exact
 *                      re-score, local winner: x[1] = binary64 bits of its
 *                      error, x[2] = row << 32 | flat bin, x[4] = kept,
 *                      x[6] = overflow (fall back to dses_stage_*)
 *                                                          -> all_reduce x[1] MIN
 *   dses_shard_key     x[2] = all-ones unless this rank holds the minimum error
 *                                                          -> all_reduce x[2] MIN
 *   dses_shard_miss    x[5] = the winner's sat_l0 miss bits on its rank, else 0
 *                                                          -> all_reduce x[3..6] SUM
 * Replaces engines.py:254-301 (M*, the q*M* cutoff, min-error / lexicographic
 * winner, candidates_evaluated / _refined, best_inliers) across ranks. */
int dses_shard_vote(dses_plan* plan, const dses_grid* grid, int64_t r_begin, int64_t r_count,
                    int64_t* xchg, void* stream);
int dses_shard_select(dses_plan* plan, double q, int metric_code, double metric_param,
                      int skip_refine, int64_t* xchg, void* stream);
int dses_shard_key(dses_plan* plan, int64_t* xchg, void* stream);
int dses_shard_miss(dses_plan* plan, int64_t* xchg, void* stream);

int dses_stage_stats(dses_plan* plan, int64_t* pairs, int64_t* votes, int64_t* rechecks);
/* Host<->device bytes and kernel launches attributed to this plan (plan
 * creation included); reset != 0 zeroes the counters after reading. */
int dses_plan_traffic(dses_plan* plan, int64_t* h2d_bytes, int64_t* d2h_bytes, int64_t* launches,
                      int reset);

/* ---- verification --------------------------------------------------------- */
/* Dense translation sweep of the mode-optimality check; replaces
 * _kernels.sweep_inlier_best (_kernels.py:384-410), called by
 * harness.run_oracle_checks (harness.py:438-440).  cands: (n*m, 3) binary64
 * differences y_j - R x_i, row-major by source i; t0/t1/t2: the lattice axes.
 * *best = max over lattice translations t of the number of sources i with
 * some j such that |cands[i*m+j] - t|_inf < half (bit-identical counts).
 * Host pointers; synchronous. */
int dses_sweep_inlier_best(int device, const double* cands, int64_t n, int64_t m, double half,
                           const double* t0, int64_t n0, const double* t1, int64_t n1,
                           const double* t2, int64_t n2, int64_t* best);

/* ---- measurement ---------------------------------------------------------- */
/* FP32 FFMA throughput of `device` measured live (independent FFMA chains on
 * every SM, CUDA events): the roofline denominator bench.py reports against. */
int dses_probe_fp32_peak(int device, double* ffma_per_s, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* DSES_B200_H */
