// dses_score.cu -- phases 2 and 3 of DSES on B200: selection and scoring.
//
// Replaces, from engines.dses (engines.py:254-285):
//   * the valid filter + stable argsort + M* (phase 2): select_stats_kernel,
//     compact_kernel (the sort order is unobservable: the winner rule is
//     order-free, engines.py:276-280, and n_score is a count);
//   * _refine_cutoff (engines.py:196-201): compact_kernel keeps
//     count >= fl(fl(q*M*) - 1e-9) in binary64, exactly as the reference;
//   * _score_poses -> refine_batch/_point_best (_kernels.py:34-80, 297-324):
//     an fp32 screen over all kept candidates (screen_kernel), then an exact
//     binary64 re-score (exact_points_kernel + exact_sum_kernel: reference
//     operation order, serial sum over i) of every candidate whose screened
//     error is within a rigorous bound of the screened minimum;
//   * the min-error / lexicographic-grid winner (winner_kernel).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdint>
#include <math_constants.h>
#include "dses_common.cuh"

namespace dses {

// Candidate counts are either host values or device counters (`dcount`,
// written by the previous kernel of the same stream): kernels loop over
// candidates with a grid stride, so a fixed grid serves either without a
// host round trip.
__device__ __forceinline__ int64_t eff_count(const unsigned long long* dcount, int64_t cap) {
  return dcount ? min((int64_t)*dcount, cap) : cap;
}


// ---------------------------------------------------------------------------
// phase 2
// ---------------------------------------------------------------------------
__global__ void select_stats_kernel(const int* counts, int64_t nrot, unsigned long long* mstar,
                                    unsigned long long* nvalid) {
  int best = 0, nv = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrot;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int c = counts[r];
    best = max(best, c);
    nv += c > 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    nv += __shfl_xor_sync(0xffffffffu, nv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(mstar, (unsigned long long)best);
    atomicAdd(nvalid, (unsigned long long)nv);
  }
}

// smallest row whose count equals mstar (the first entry of the stable order)
__global__ void argmax_kernel(const int* counts, int64_t nrot, int64_t r_begin, int mstar,
                              unsigned long long* row, const unsigned long long* dmstar) {
  if (dmstar) mstar = (int)*dmstar;
  unsigned long long best = ULLONG_MAX;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrot;
       r += (int64_t)gridDim.x * blockDim.x)
    if (counts[r] == mstar && mstar > 0) best = min(best, (unsigned long long)(r + r_begin));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != ULLONG_MAX) atomicMin(row, best);
}

__global__ void compact_kernel(const int* counts, const int* lins, int64_t nrot, int64_t r_begin,
                               double cutoff, int64_t* rows, int* cand_lins,
                               unsigned long long* ncand, const unsigned long long* dmstar,
                               double q) {
  // engines.py:196-201 in binary64: cutoff = q * M* - 1e-9 (M* on the device
  // when dmstar is given)
  // explicit roundings: nvcc would otherwise contract this into one DFMA
  if (dmstar) cutoff = dsub(dmul(q, (double)*dmstar), 1e-9);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrot;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int c = counts[r];
    const bool keep = c > 0 && (double)c >= cutoff;
    const unsigned m = __ballot_sync(__activemask(), keep);
    if (!m) continue;
    // warp-aggregated slot reservation
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(ncand, (unsigned long long)__popc(m));
    base = __shfl_sync(m | (1u << leader), base, leader);
    if (keep) {
      const int k = (int)base + __popc(m & ((1u << lane) - 1));
      rows[k] = r + r_begin;
      cand_lins[k] = lins[r];
    }
  }
}

// ---------------------------------------------------------------------------
// pose helpers
// ---------------------------------------------------------------------------
// t = bin_center(_decode_flat(lin)) = (f + ilo) * bin  (mode_search.py:51-54,167-171)
__device__ __forceinline__ void decode_translation(const ScoreParams& s, int lin, double* t) {
  const int a = lin / (s.d1 * s.d2), rem = lin % (s.d1 * s.d2), b = rem / s.d2, c = rem % s.d2;
  if (s.exh_k >= 0) {  // t_center + side * trans_bin, side = -k..k (engines.py:168-169)
    t[0] = dadd(s.tcen[0], dmul((double)(a - s.exh_k), s.bin_size));
    t[1] = dadd(s.tcen[1], dmul((double)(b - s.exh_k), s.bin_size));
    t[2] = dadd(s.tcen[2], dmul((double)(c - s.exh_k), s.bin_size));
    return;
  }
  t[0] = dmul((double)(a + s.ilo0), s.bin_size);
  t[1] = dmul((double)(b + s.ilo1), s.bin_size);
  t[2] = dmul((double)(c + s.ilo2), s.bin_size);
}

// p = ((r0 x0 + r1 x1) + r2 x2) + t  (_kernels.py:320-322)
__device__ __forceinline__ void pose_point(const double* R, const double* t, const double* x,
                                           double* pp) {
#pragma unroll
  for (int k = 0; k < 3; ++k) pp[k] = dadd(rot_row(R, k, x[0], x[1], x[2]), t[k]);
}

__device__ __forceinline__ int lower_bound_d(const double* a, int n, double v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// _point_best (_kernels.py:34-80) in binary64, reference semantics (windows
// over the axis-0-sorted reference, strict sat_l0 test), plus code 4.
__device__ double exact_point_best(const ScoreParams& s, double p0, double p1, double p2) {
  const double* y0 = s.ys0;
  const double* y1 = s.ys1;
  const double* y2 = s.ys2;
  const int m = s.m;
  if (s.code == kTruncL1 || s.code == kTruncL2) {
    const double lo = dsub(p0, s.param), hi = dadd(p0, s.param);
    const int jlo = lower_bound_d(y0, m, lo);
    const int jhi = lower_bound_d(y0, m, hi);
    // The reference scans the axis-0 window [lo, hi) (jlo..jhi in axis-0
    // order).  When that slab is wide (surfaces perpendicular to axis 0),
    // visit instead the uniform-grid cells around the tau-box: the same
    // window test and the same binary64 distance per point, so the minimum
    // is identical -- a point with |y_k - p_k| > tau on axis 1 or 2 has a
    // distance >= tau (monotone rounding) and cannot lower best = tau.
    int cl[3], ch[3];
    int ncell = 1;
    const double pk[3] = {p0, p1, p2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cl[k] = max(0, __float2int_rd(((float)dsub(pk[k], s.param) - s.gorg[k]) * s.ginv) - 1);
      ch[k] = min(s.gdim[k] - 1, __float2int_rd(((float)dadd(pk[k], s.param) - s.gorg[k]) * s.ginv) + 1);
      ncell *= max(0, ch[k] - cl[k] + 1);
    }
    if ((float)(jhi - jlo) > 2.0f * (float)ncell * (1.0f + s.gppc)) {
      const double cap = s.code == kTruncL1 ? s.param : dmul(s.param, s.param);
      double best = cap;
      for (int x = cl[0]; x <= ch[0]; ++x)
        for (int yy = cl[1]; yy <= ch[1]; ++yy)
          for (int z = cl[2]; z <= ch[2]; ++z) {
            const int2 rg = __ldg(&s.gcell[(x * s.gdim[1] + yy) * s.gdim[2] + z]);
            for (int q = rg.x; q < rg.y; ++q) {
              const int j = __float_as_int(__ldg(&s.gpts[q]).w);
              const double yj0 = y0[j];
              if (!(yj0 >= lo && yj0 < hi)) continue;  // the reference's window
              double v;
              if (s.code == kTruncL1) {
                v = dadd(dadd(fabs(dsub(yj0, p0)), fabs(dsub(y1[j], p1))), fabs(dsub(y2[j], p2)));
              } else {
                const double a = dsub(yj0, p0), b = dsub(y1[j], p1), c = dsub(y2[j], p2);
                v = dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c));
              }
              if (v < best) best = v;
            }
          }
      if (s.code == kTruncL1) return best;
      return best < cap ? sqrt(best) : s.param;
    }
    if (s.code == kTruncL1) {
      double best = s.param;
      for (int j = jlo; j < jhi; ++j) {
        const double v = dadd(dadd(fabs(dsub(y0[j], p0)), fabs(dsub(y1[j], p1))), fabs(dsub(y2[j], p2)));
        if (v < best) best = v;
      }
      return best;
    }
    const double cap = dmul(s.param, s.param);
    double best = cap;
    for (int j = jlo; j < jhi; ++j) {
      const double a = dsub(y0[j], p0), b = dsub(y1[j], p1), c = dsub(y2[j], p2);
      const double v = dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c));
      if (v < best) best = v;
    }
    return best < cap ? sqrt(best) : s.param;
  }
  if (s.code == kSatL0) {
    const double half = dmul(0.5, s.param);
    const int jlo = lower_bound_d(y0, m, dsub(p0, half));
    const int jhi = lower_bound_d(y0, m, dadd(p0, half));
    for (int j = jlo; j < jhi; ++j)
      if (fabs(dsub(y0[j], p0)) < half && fabs(dsub(y1[j], p1)) < half && fabs(dsub(y2[j], p2)) < half)
        return 0.0;
    return 1.0;
  }
  double best = CUDART_INF;
  if (s.code == kL1) {
    for (int j = 0; j < m; ++j) {
      const double v = dadd(dadd(fabs(dsub(y0[j], p0)), fabs(dsub(y1[j], p1))), fabs(dsub(y2[j], p2)));
      if (v < best) best = v;
    }
    return best;
  }
  for (int j = 0; j < m; ++j) {
    const double a = dsub(y0[j], p0), b = dsub(y1[j], p1), c = dsub(y2[j], p2);
    const double v = dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c));
    if (v < best) best = v;
  }
  return sqrt(best);
}

__device__ __forceinline__ void load_pose(const ScoreParams& s, int64_t row, int lin, double* R,
                                          double* t) {
  if (threadIdx.x < 9) R[threadIdx.x] = rotation_entry(s.rot, row, threadIdx.x);
  if (threadIdx.x == 0) {
    if (s.tvec) { t[0] = s.tvec[3 * row]; t[1] = s.tvec[3 * row + 1]; t[2] = s.tvec[3 * row + 2]; }
    else decode_translation(s, lin, t);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// phase 3a: fp32 screen.  grid (ceil(n/kScreenThreads), ncand); one source
// point per thread; the reference cloud streams through shared memory in
// chunks (broadcast reads).  For windowed metrics the block only visits the
// reference slice whose axis-0 coordinate can fall inside some thread's window.
// ---------------------------------------------------------------------------
constexpr int kScreenThreads = 256;
constexpr int kScreenChunk = 2048;  // reference points per shared-memory chunk (32 KB)

__global__ void __launch_bounds__(kScreenThreads) screen_kernel(ScoreParams s, const int64_t* rows,
                                                                const int* lins, double* partial,
                                                                const unsigned long long* dcount,
                                                                int64_t ncand) {
  __shared__ double R[9], t[3];
  __shared__ float4 ych[kScreenChunk];
  __shared__ float wred[2][kScreenThreads / 32];
  __shared__ int jrange[2];
  __shared__ double sred[kScreenThreads / 32];
  const int64_t nc = eff_count(dcount, ncand);
  for (int64_t c = blockIdx.y; c < nc; c += gridDim.y) {
  load_pose(s, rows[c], lins[c], R, t);
  const int i = blockIdx.x * kScreenThreads + threadIdx.x;
  const bool active = i < s.n;
  double pp[3] = {0.0, 0.0, 0.0};
  if (active) pose_point(R, t, s.x + 3 * i, pp);
  const float p0 = (float)pp[0], p1 = (float)pp[1], p2 = (float)pp[2];
  const bool windowed = (s.code == kTruncL1 || s.code == kTruncL2 || s.code == kSatL0);
  const float wr = s.code == kSatL0 ? s.halff : s.paramf;
  int jlo = 0, jhi = s.m;
  if (windowed) {
    float lo = active ? p0 : FLT_MAX, hi = active ? p0 : -FLT_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) { wred[0][threadIdx.x >> 5] = lo; wred[1][threadIdx.x >> 5] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      lo = wred[0][0]; hi = wred[1][0];
      for (int w = 1; w < kScreenThreads / 32; ++w) { lo = fminf(lo, wred[0][w]); hi = fmaxf(hi, wred[1][w]); }
      // widen by the window and an fp32 slack; the exact re-score uses exact windows
      const double slack = 1e-5 * (1.0 + fabs((double)lo) + fabs((double)hi)) + s.amb;
      jrange[0] = lower_bound_d(s.ys0, s.m, (double)lo - (double)wr - slack);
      jrange[1] = lower_bound_d(s.ys0, s.m, (double)hi + (double)wr + slack);
    }
    __syncthreads();
    jlo = jrange[0];
    jhi = jrange[1];
  }
  float best = FLT_MAX;
  bool inlier = false, ambiguous = false;
  const float half = s.halff, amb = s.amb;
  for (int base = jlo; base < jhi; base += kScreenChunk) {
    const int cnt = min(kScreenChunk, jhi - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kScreenThreads) ych[k] = s.ysf[base + k];
    __syncthreads();
    if (s.code == kL1 || s.code == kTruncL1) {
#pragma unroll 8
      for (int k = 0; k < cnt; ++k) {
        const float4 y = ych[k];
        best = fminf(best, fabsf(y.x - p0) + fabsf(y.y - p1) + fabsf(y.z - p2));
      }
    } else if (s.code == kL2 || s.code == kTruncL2) {
#pragma unroll 8
      for (int k = 0; k < cnt; ++k) {
        const float4 y = ych[k];
        const float a = y.x - p0, b = y.y - p1, d = y.z - p2;
        best = fminf(best, fmaf(d, d, fmaf(b, b, a * a)));
      }
    } else {
      for (int k = 0; k < cnt; ++k) {
        const float4 y = ych[k];
        const float m = fmaxf(fmaxf(fabsf(y.x - p0), fabsf(y.y - p1)), fabsf(y.z - p2));
        inlier |= m < half - amb;
        ambiguous |= m < half + amb;
      }
    }
  }
  double v = 0.0;
  if (active) {
    if (s.code == kL1) v = best;
    else if (s.code == kTruncL1) v = fminf(best, s.paramf);
    else if (s.code == kL2) v = sqrtf(best);
    else if (s.code == kTruncL2) v = fminf(sqrtf(best), s.paramf);
    else v = inlier ? 0.0 : (ambiguous ? exact_point_best(s, pp[0], pp[1], pp[2]) : 1.0);
  }
  // deterministic block sum in binary64
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kScreenThreads / 32; ++w) tot += sred[w];
    partial[(size_t)c * gridDim.x + blockIdx.x] = tot;
  }
  __syncthreads();  // shared pose / chunk / reduction reused by the next candidate
  }
}

// ---------------------------------------------------------------------------
// phase 3a (grid): fp32 screen with uniform-grid nearest-neighbour lookups
// into the full reference cloud (used for truncated L1 / L2; the kernel also
// handles L1 / L2).  Per source
// point, shells of cells at Chebyshev radius r = 0, 1, 2, ... around the
// point's (clamped) cell are visited until the best distance is provably
// below every unvisited point: a point outside the shells 0..r-1 differs
// from the query by >= (r-1) h along some axis, so the search stops once
// best <= (r-1) h (scaled down by 1e-6 against fp32 rounding).  Truncated
// metrics start from best = tau, so they visit only shells within tau.
// Beyond radius kGridShells the point falls back to a full scan.
// ---------------------------------------------------------------------------
constexpr int kGridShells = 4;

template <bool L2>
__device__ __forceinline__ float cell_scan(const ScoreParams& s, int cell, float p0, float p1, float p2,
                                           float best) {
  const int2 rg = __ldg(&s.gcell[cell]);
  for (int q = rg.x; q < rg.y; ++q) {
    const float4 y = __ldg(&s.gpts[q]);
    const float a = y.x - p0, b = y.y - p1, d = y.z - p2;
    best = fminf(best, L2 ? fmaf(d, d, fmaf(b, b, a * a)) : fabsf(a) + fabsf(b) + fabsf(d));
  }
  return best;
}

template <bool L2>
__device__ float grid_nn(const ScoreParams& s, float p0, float p1, float p2, float best) {
  const float pc[3] = {p0, p1, p2};
  int c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
    c[k] = min(s.gdim[k] - 1, max(0, __float2int_rd((pc[k] - s.gorg[k]) * s.ginv)));
  const int rmax = max(s.gdim[0], max(s.gdim[1], s.gdim[2]));
  for (int r = 0; r <= rmax; ++r) {
    if (r > 0) {
      const float lb = (float)(r - 1) * s.gh * (1.0f - 1e-6f);
      if ((L2 ? lb * lb : lb) >= best) break;
    }
    if (r > kGridShells) {  // far from the cloud: full scan
      for (int q = 0; q < s.m; ++q) {
        const float4 y = __ldg(&s.gpts[q]);
        const float a = y.x - p0, b = y.y - p1, d = y.z - p2;
        best = fminf(best, L2 ? fmaf(d, d, fmaf(b, b, a * a)) : fabsf(a) + fabsf(b) + fabsf(d));
      }
      break;
    }
    for (int dx = -r; dx <= r; ++dx) {
      const int x = c[0] + dx;
      if (x < 0 || x >= s.gdim[0]) continue;
      for (int dy = -r; dy <= r; ++dy) {
        const int yy = c[1] + dy;
        if (yy < 0 || yy >= s.gdim[1]) continue;
        const bool edge = (dx == -r) | (dx == r) | (dy == -r) | (dy == r);
        const int step = edge ? 1 : max(1, 2 * r);
        for (int dz = -r; dz <= r; dz += step) {
          const int z = c[2] + dz;
          if (z < 0 || z >= s.gdim[2]) continue;
          best = cell_scan<L2>(s, (x * s.gdim[1] + yy) * s.gdim[2] + z, p0, p1, p2, best);
        }
      }
    }
  }
  return best;
}

__global__ void __launch_bounds__(kScreenThreads) screen_grid_kernel(ScoreParams s, const int64_t* rows,
                                                                     const int* lins, double* partial,
                                                                     const unsigned long long* dcount,
                                                                     int64_t ncand) {
  __shared__ double R[9], t[3];
  __shared__ double sred[kScreenThreads / 32];
  const int64_t nc = eff_count(dcount, ncand);
  for (int64_t c = blockIdx.y; c < nc; c += gridDim.y) {
  load_pose(s, rows[c], lins[c], R, t);
  const int i = blockIdx.x * kScreenThreads + threadIdx.x;
  double v = 0.0;
  if (i < s.n) {
    double pp[3];
    pose_point(R, t, s.x + 3 * i, pp);
    const float p0 = (float)pp[0], p1 = (float)pp[1], p2 = (float)pp[2];
    if (s.code == kL1) v = grid_nn<false>(s, p0, p1, p2, FLT_MAX);
    else if (s.code == kTruncL1) v = grid_nn<false>(s, p0, p1, p2, s.paramf);
    else if (s.code == kL2) v = sqrtf(grid_nn<true>(s, p0, p1, p2, FLT_MAX));
    else v = fminf(sqrtf(grid_nn<true>(s, p0, p1, p2, s.paramf * s.paramf)), s.paramf);
  }
  // deterministic block sum in binary64
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < kScreenThreads / 32; ++w) tot += sred[w];
    partial[(size_t)c * gridDim.x + blockIdx.x] = tot;
  }
  __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// phase 3a (full scan, L1 / L2): kScanCands candidates per block share every
// reference point read from shared memory (register blocking: one broadcast
// LDS feeds kScanCands distance evaluations).
// ---------------------------------------------------------------------------
constexpr int kScanCands = 4;
#ifndef DSES_SCAN_F32X2
#define DSES_SCAN_F32X2 1
#endif
// f32x2 helpers (sm_100 packed single precision)
__device__ __forceinline__ unsigned long long pack_f2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack_f2(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long sub_f2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long mul_f2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long fma_f2(unsigned long long a, unsigned long long b,
                                                     unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

template <bool L2>
__global__ void __launch_bounds__(kScreenThreads) screen_scan_kernel(ScoreParams s, const int64_t* rows,
                                                                     const int* lins, int64_t ncand_cap,
                                                                     double* partial,
                                                                     const unsigned long long* dcount) {
  __shared__ double R[kScanCands][9], t[kScanCands][3];
  __shared__ float4 ych[kScreenChunk];
  __shared__ double sred[kScanCands][kScreenThreads / 32];
  const int64_t ncand = eff_count(dcount, ncand_cap);
  const int64_t ngroups = (ncand + kScanCands - 1) / kScanCands;
  for (int64_t g = blockIdx.y; g < ngroups; g += gridDim.y) {
  const int64_t c0 = g * kScanCands;
  for (int q = 0; q < kScanCands; ++q) {
    const int64_t c = min(c0 + q, ncand - 1);
    if (threadIdx.x < 9) R[q][threadIdx.x] = rotation_entry(s.rot, rows[c], threadIdx.x);
    if (threadIdx.x == 0) {
      if (s.tvec) { t[q][0] = s.tvec[3 * rows[c]]; t[q][1] = s.tvec[3 * rows[c] + 1]; t[q][2] = s.tvec[3 * rows[c] + 2]; }
      else decode_translation(s, lins[c], t[q]);
    }
  }
  __syncthreads();
  const int i = blockIdx.x * kScreenThreads + threadIdx.x;
  const bool active = i < s.n;
  float px[kScanCands], py[kScanCands], pz[kScanCands], best[kScanCands];
#pragma unroll
  for (int q = 0; q < kScanCands; ++q) {
    double pp[3] = {0.0, 0.0, 0.0};
    if (active) pose_point(R[q], t[q], s.x + 3 * i, pp);
    px[q] = (float)pp[0]; py[q] = (float)pp[1]; pz[q] = (float)pp[2];
    best[q] = FLT_MAX;
  }
  for (int base = 0; base < s.m; base += kScreenChunk) {
    const int cnt = min(kScreenChunk, s.m - base);
    __syncthreads();
    for (int k = threadIdx.x; k < cnt; k += kScreenThreads) ych[k] = s.ysf[base + k];
    __syncthreads();
#if DSES_SCAN_F32X2
    // candidate pairs packed in f32x2 registers (FADD2 / FMUL2 / FFMA2: one
    // instruction per two candidates, same IEEE rounding as the scalar ops)
    unsigned long long PX[kScanCands / 2], PY[kScanCands / 2], PZ[kScanCands / 2];
#pragma unroll
    for (int h = 0; h < kScanCands / 2; ++h) {
      PX[h] = pack_f2(px[2 * h], px[2 * h + 1]);
      PY[h] = pack_f2(py[2 * h], py[2 * h + 1]);
      PZ[h] = pack_f2(pz[2 * h], pz[2 * h + 1]);
    }
#pragma unroll 4
    for (int k = 0; k < cnt; ++k) {
      const float4 y = ych[k];
      const unsigned long long yx = pack_f2(y.x, y.x), yy = pack_f2(y.y, y.y), yz = pack_f2(y.z, y.z);
#pragma unroll
      for (int h = 0; h < kScanCands / 2; ++h) {
        const unsigned long long a = sub_f2(yx, PX[h]), b = sub_f2(yy, PY[h]), d = sub_f2(yz, PZ[h]);
        float lo, hi;
        if (L2) {
          unpack_f2(fma_f2(d, d, fma_f2(b, b, mul_f2(a, a))), lo, hi);
        } else {
          float a0, a1, b0, b1, d0, d1;
          unpack_f2(a, a0, a1);
          unpack_f2(b, b0, b1);
          unpack_f2(d, d0, d1);
          lo = fabsf(a0) + fabsf(b0) + fabsf(d0);
          hi = fabsf(a1) + fabsf(b1) + fabsf(d1);
        }
        best[2 * h] = fminf(best[2 * h], lo);
        best[2 * h + 1] = fminf(best[2 * h + 1], hi);
      }
    }
#else
#pragma unroll 4
    for (int k = 0; k < cnt; ++k) {
      const float4 y = ych[k];
#pragma unroll
      for (int q = 0; q < kScanCands; ++q) {
        const float a = y.x - px[q], b = y.y - py[q], d = y.z - pz[q];
        best[q] = fminf(best[q], L2 ? fmaf(d, d, fmaf(b, b, a * a)) : fabsf(a) + fabsf(b) + fabsf(d));
      }
    }
#endif
  }
#pragma unroll
  for (int q = 0; q < kScanCands; ++q) {
    double v = active ? (L2 ? sqrtf(best[q]) : best[q]) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sred[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < kScanCands && c0 + threadIdx.x < ncand) {
    double tot = 0.0;
    for (int w = 0; w < kScreenThreads / 32; ++w) tot += sred[threadIdx.x][w];
    partial[(size_t)(c0 + threadIdx.x) * gridDim.x + blockIdx.x] = tot;
  }
  __syncthreads();
  }
}

// err32[c] = sum of the block partials in block order; atomicMin of the
// (non-negative) binary64 bits gives the minimum.
__global__ void screen_reduce_kernel(const double* partial, int nblk, int64_t ncand, double* err,
                                     unsigned long long* minbits, const unsigned long long* dcount) {
  const int64_t nc = eff_count(dcount, ncand);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x) {
    double tot = 0.0;
    for (int b = 0; b < nblk; ++b) tot += partial[c * nblk + b];
    err[c] = tot;
    atomicMin(minbits, (unsigned long long)__double_as_longlong(tot));
  }
}

// keep candidates with screened error <= threshold; with `dmin` the
// threshold is (device minimum) + tol
__global__ void rescore_compact_kernel(const double* err, int64_t ncand, double threshold,
                                       int* sel, unsigned long long* nsel,
                                       const unsigned long long* dcount,
                                       const unsigned long long* dmin, double tol) {
  const int64_t nc = eff_count(dcount, ncand);
  const double thr = dmin ? __longlong_as_double((long long)*dmin) + tol : threshold;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc;
       c += (int64_t)gridDim.x * blockDim.x)
    if (err[c] <= thr) sel[atomicAdd(nsel, 1ull)] = (int)c;
}

// ---------------------------------------------------------------------------
// phase 3b: exact binary64 re-score, reference semantics and operation order.
// grid (ceil(n/128), nsel): per-point values; then one thread per candidate
// sums them serially in source order (_kernels.py:315-324).
// ---------------------------------------------------------------------------
// One warp per (candidate, source point): _point_best (_kernels.py:34-80)
// with the scan split over the lanes.  Each lane evaluates a subset of the
// same points with the same binary64 operations as exact_point_best; the
// minimum (and sat_l0's "any inlier") is order-independent, so the warp
// reduction gives the identical value.  The points scanned are the
// reference's own window (axis-0-sorted, [p0 - tau, p0 + tau) / half-width
// for sat_l0), or -- when that slab is wide, e.g. a surface perpendicular to
// axis 0 -- the uniform-grid cells around the (tau-)box with the same window
// test per point (a point outside the box on axis 1 or 2 cannot lower the
// truncated minimum, resp. cannot be a strict Chebyshev inlier).
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ double exact_point_best_warp(const ScoreParams& s, double p0, double p1, double p2,
                                        int lane) {
  const double* y0 = s.ys0;
  const double* y1 = s.ys1;
  const double* y2 = s.ys2;
  const int m = s.m;
  if (s.code == kL1 || s.code == kL2) {  // every reference point
    double best = CUDART_INF;
    for (int j = lane; j < m; j += 32) {
      double v;
      if (s.code == kL1) {
        v = dadd(dadd(fabs(dsub(y0[j], p0)), fabs(dsub(y1[j], p1))), fabs(dsub(y2[j], p2)));
      } else {
        const double a = dsub(y0[j], p0), b = dsub(y1[j], p1), c = dsub(y2[j], p2);
        v = dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c));
      }
      if (v < best) best = v;
    }
    best = warp_min_d(best);
    return s.code == kL1 ? best : sqrt(best);
  }
  const bool sat = s.code == kSatL0;
  const double w = sat ? dmul(0.5, s.param) : s.param;   // window half-width
  const double lo = dsub(p0, w), hi = dadd(p0, w);
  const int jlo = lower_bound_d(y0, m, lo);
  const int jhi = lower_bound_d(y0, m, hi);
  const double cap = sat ? 1.0 : (s.code == kTruncL1 ? s.param : dmul(s.param, s.param));
  double best = cap;
  bool hit = false;
  // the lane's point j: the truncated distance / strict inlier test
  auto visit = [&](int j) {
    const double yj0 = y0[j];
    if (sat) {
      hit |= fabs(dsub(yj0, p0)) < w && fabs(dsub(y1[j], p1)) < w && fabs(dsub(y2[j], p2)) < w;
      return;
    }
    double v;
    if (s.code == kTruncL1) {
      v = dadd(dadd(fabs(dsub(yj0, p0)), fabs(dsub(y1[j], p1))), fabs(dsub(y2[j], p2)));
    } else {
      const double a = dsub(yj0, p0), b = dsub(y1[j], p1), c = dsub(y2[j], p2);
      v = dadd(dadd(dmul(a, a), dmul(b, b)), dmul(c, c));
    }
    if (v < best) best = v;
  };
  int cl[3], ch[3];
  int ncell = 1;
  const double pk[3] = {p0, p1, p2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    cl[k] = max(0, __float2int_rd(((float)dsub(pk[k], w) - s.gorg[k]) * s.ginv) - 1);
    ch[k] = min(s.gdim[k] - 1, __float2int_rd(((float)dadd(pk[k], w) - s.gorg[k]) * s.ginv) + 1);
    ncell *= max(0, ch[k] - cl[k] + 1);
  }
  if ((float)(jhi - jlo) > 2.0f * (float)ncell * (1.0f + s.gppc)) {
    const int ny = ch[1] - cl[1] + 1, nz = ch[2] - cl[2] + 1;
    for (int t = lane; t < ncell; t += 32) {  // lane = cell of the box
      const int x = cl[0] + t / (ny * nz), yy = cl[1] + (t / nz) % ny, z = cl[2] + t % nz;
      const int2 rg = __ldg(&s.gcell[(x * s.gdim[1] + yy) * s.gdim[2] + z]);
      for (int q = rg.x; q < rg.y; ++q) {
        const int j = __float_as_int(__ldg(&s.gpts[q]).w);
        const double yj0 = y0[j];
        if (yj0 >= lo && yj0 < hi) visit(j);  // the reference's window
      }
    }
  } else {
    for (int j = jlo + lane; j < jhi; j += 32) visit(j);
  }
  if (sat) return __any_sync(0xffffffffu, hit) ? 0.0 : 1.0;
  best = warp_min_d(best);
  if (s.code == kTruncL1) return best;
  return best < cap ? sqrt(best) : s.param;
}

constexpr int kExactThreads = 128;

// warp = source point (kExactThreads / 32 points per block), y = candidate
__global__ void __launch_bounds__(kExactThreads) exact_points_kernel(ScoreParams s,
                                                                     const int64_t* rows,
                                                                     const int* lins,
                                                                     const int* sel, int64_t nsel_cap,
                                                                     double* vals,
                                                                     const unsigned long long* dcount) {
  __shared__ double R[9], t[3];
  const int64_t nsel = eff_count(dcount, nsel_cap);
  const int lane = threadIdx.x & 31;
  for (int64_t k = blockIdx.y; k < nsel; k += gridDim.y) {
    const int64_t c = sel ? sel[k] : k;
    if (c < 0) continue;  // no winner (block-uniform)
    load_pose(s, rows[c], lins[c], R, t);
    const int i = blockIdx.x * (kExactThreads / 32) + (threadIdx.x >> 5);
    if (i < s.n) {  // warp-uniform
      double pp[3];
      pose_point(R, t, s.x + 3 * i, pp);
      const double v = exact_point_best_warp(s, pp[0], pp[1], pp[2], lane);
      if (lane == 0) vals[(size_t)k * s.n + i] = v;
    }
    __syncthreads();
  }
}

// The serial binary64 sum over i in the reference's order
// (_kernels.py:297-324: err += point_best, i = 0..n-1).  One warp per
// candidate: lanes load 32 consecutive values (coalesced, in flight
// together), lane 0 adds them in order as they arrive by shuffle -- the same
// dependent chain of additions, without a global-load latency per term.
// `integral`: the terms are 0.0 / 1.0 (sat_l0), so every summation order
// gives the same (exact, integer) total and the lanes reduce in parallel.
__global__ void exact_sum_kernel(const double* vals, int n, int64_t nsel_cap, double* out,
                                 const unsigned long long* dcount, bool integral) {
  const int64_t nsel = eff_count(dcount, nsel_cap);
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < nsel; c += warps) {
    const double* v = vals + (size_t)c * n;
    if (integral) {
      double part = 0.0;
      for (int i = lane; i < n; i += 32) part += v[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) out[c] = part;
      continue;
    }
    double total = 0.0;
    int i0 = 0;
    // full chunks: the next chunk's load and the shuffles are issued ahead of
    // the dependent adds (the serial chain is then DADD latency, not memory)
    double next = n >= 32 ? v[lane] : 0.0;
    for (; i0 + 32 <= n; i0 += 32) {
      const double mine = next;
      if (i0 + 64 <= n) next = v[i0 + 32 + lane];
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = __shfl_sync(0xffffffffu, mine, k0 + k);
#pragma unroll
        for (int k = 0; k < 8; ++k) total = dadd(total, t[k]);
      }
    }
    if (i0 < n) {
      const double mine = i0 + lane < n ? v[i0 + lane] : 0.0;
      for (int k = 0; k < n - i0; ++k) total = dadd(total, __shfl_sync(0xffffffffu, mine, k));
    }
    if (lane == 0) out[c] = total;
  }
}

// lexicographic (error, row) minimum over the re-scored set; single block.
__global__ void winner_kernel(const double* err64, const int* sel, const int64_t* rows,
                              int64_t nsel_cap, double* best_err, int64_t* best_row, int* best_c,
                              const int* lins, const unsigned long long* dcount) {
  const int64_t nsel = eff_count(dcount, nsel_cap);
  __shared__ double se[32];
  __shared__ int64_t sr[32];
  __shared__ int sc[32];
  double e = CUDART_INF;
  int64_t r = INT64_MAX;
  int cc = -1;
  for (int64_t k = threadIdx.x; k < nsel; k += blockDim.x) {
    const int c = sel ? sel[k] : (int)k;
    const double ek = err64[k];
    // tie-break key: the flat rotation index (lexicographic grid order,
    // engines.py:276-280); with `lins` (exhaustive search) rotation-major then
    // translation index, i.e. the pose enumeration order (_kernels.py:327-381)
    const int64_t rk = lins ? rows[c] * ((int64_t)1 << 31) + lins[c] : rows[c];
    if (ek < e || (ek == e && rk < r)) { e = ek; r = rk; cc = c; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double oe = __shfl_xor_sync(0xffffffffu, e, o);
    const int64_t orr = __shfl_xor_sync(0xffffffffu, r, o);
    const int oc = __shfl_xor_sync(0xffffffffu, cc, o);
    if (oe < e || (oe == e && orr < r)) { e = oe; r = orr; cc = oc; }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { se[w] = e; sr[w] = r; sc[w] = cc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    e = se[0]; r = sr[0]; cc = sc[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (se[k] < e || (se[k] == e && sr[k] < r)) { e = se[k]; r = sr[k]; cc = sc[k]; }
    *best_err = e;
    *best_row = lins ? (cc >= 0 ? rows[cc] : INT64_MAX) : r;
    *best_c = cc;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int screen_threads() { return kScreenThreads; }
int exact_threads() { return kExactThreads; }

cudaError_t launch_select_stats(const int* counts, int64_t nrot, unsigned long long* mstar,
                                unsigned long long* nvalid, int sms, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((nrot + 255) / 256, (int64_t)sms * 8);
  select_stats_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(counts, nrot, mstar, nvalid);
  return cudaGetLastError();
}

cudaError_t launch_argmax(const int* counts, int64_t nrot, int64_t r_begin, int mstar,
                          unsigned long long* row, int sms, cudaStream_t st,
                          const unsigned long long* dmstar) {
  const int grid = (int)std::min<int64_t>((nrot + 255) / 256, (int64_t)sms * 8);
  argmax_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(counts, nrot, r_begin, mstar, row, dmstar);
  return cudaGetLastError();
}

cudaError_t launch_compact(const int* counts, const int* lins, int64_t nrot, int64_t r_begin,
                           double cutoff, int64_t* rows, int* cl, unsigned long long* ncand, int sms,
                           cudaStream_t st, const unsigned long long* dmstar, double q) {
  const int grid = (int)std::min<int64_t>((nrot + 255) / 256, (int64_t)sms * 8);
  compact_kernel<<<grid > 0 ? grid : 1, 256, 0, st>>>(counts, lins, nrot, r_begin, cutoff, rows, cl,
                                                      ncand, dmstar, q);
  return cudaGetLastError();
}

// `ncand` is the exact count (dcount == nullptr) or an upper bound of the
// device counter *dcount; the grid is capped (candidate-strided kernels).
cudaError_t launch_screen(const ScoreParams& s, const int64_t* rows, const int* lins,
                          int64_t ncand, double* partial, double* err,
                          unsigned long long* minbits, cudaStream_t st,
                          const unsigned long long* dcount) {
  if (ncand <= 0) return cudaSuccess;
  const int nblk = (s.n + kScreenThreads - 1) / kScreenThreads;
  const int64_t cap_y = std::max<int64_t>(1, std::min<int64_t>(65535, 4096 / nblk));
  if (s.code == kL1 || s.code == kL2) {
    const int64_t ng = (ncand + kScanCands - 1) / kScanCands;
    const dim3 grid(nblk, (unsigned)std::min<int64_t>(ng, dcount ? cap_y : 65535));
    if (s.code == kL1)
      screen_scan_kernel<false><<<grid, kScreenThreads, 0, st>>>(s, rows, lins, ncand, partial, dcount);
    else
      screen_scan_kernel<true><<<grid, kScreenThreads, 0, st>>>(s, rows, lins, ncand, partial, dcount);
  } else {
    // truncated metrics: grid lookups bounded by tau; L1 / L2 (unbounded
    // nearest neighbour, far points in poorly aligned candidates) and sat_l0
    // keep the streamed full / windowed scan, measured faster for them
    const dim3 grid(nblk, (unsigned)std::min<int64_t>(ncand, dcount ? cap_y : 65535));
    if (s.code != kTruncL1 && s.code != kTruncL2)
      screen_kernel<<<grid, kScreenThreads, 0, st>>>(s, rows, lins, partial, dcount, ncand);
    else
      screen_grid_kernel<<<grid, kScreenThreads, 0, st>>>(s, rows, lins, partial, dcount, ncand);
  }
  const int rb = (int)std::min<int64_t>(dcount ? 256 : 65535, (ncand + 255) / 256);
  screen_reduce_kernel<<<std::max(rb, 1), 256, 0, st>>>(partial, nblk, ncand, err, minbits, dcount);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// single-GPU search tail without host round trips (dses_search)
// ---------------------------------------------------------------------------
// sat_l0 shortcut winner (engines.py:265-268): the argmax row becomes
// candidate 0 so the inlier pass below reads it like a re-scored winner
__global__ void pick_argmax_kernel(const unsigned long long* row, const int* lins, int64_t r_begin,
                                   int64_t* cand_rows, int* cand_lins, int* win_c) {
  const unsigned long long r = *row;
  if (r == ~0ull) { cand_rows[0] = 0; cand_lins[0] = 0; *win_c = -1; return; }
  cand_rows[0] = (int64_t)r;
  cand_lins[0] = lins[(int64_t)r - r_begin];
  *win_c = 0;
}

// result record: [0] mstar [1] nvalid [2] kept [3] nsel [4] winner row [5] winner lin
// [6] winner count [7] pairs [8] votes [9] rechecks, doubles: [10] best error [11] miss
__global__ void finalize_kernel(const unsigned long long* scal, const double* win_err,
                                const int* win_c, const int64_t* cand_rows, const int* cand_lins,
                                const int* counts, int64_t r_begin, const double* miss,
                                unsigned long long* stats, long long* rec) {
  rec[0] = (long long)scal[0];
  rec[1] = (long long)scal[1];
  rec[2] = (long long)scal[3];
  rec[3] = (long long)scal[5];
  const int c = *win_c;
  const int64_t row = c >= 0 ? cand_rows[c] : -1;
  rec[4] = row;
  rec[5] = c >= 0 ? cand_lins[c] : -1;
  rec[6] = c >= 0 ? counts[row - r_begin] : 0;
  rec[7] = (long long)stats[0];
  rec[8] = (long long)stats[1];
  rec[9] = (long long)stats[2];
  stats[0] = stats[1] = stats[2] = 0;
  reinterpret_cast<double*>(rec)[10] = c >= 0 ? *win_err : 0.0;
  reinterpret_cast<double*>(rec)[11] = c >= 0 ? *miss : 0.0;
}

cudaError_t launch_pick_argmax(const unsigned long long* row, const int* lins, int64_t r_begin,
                               int64_t* cand_rows, int* cand_lins, int* win_c, cudaStream_t st) {
  pick_argmax_kernel<<<1, 1, 0, st>>>(row, lins, r_begin, cand_rows, cand_lins, win_c);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const unsigned long long* scal, const double* win_err, const int* win_c,
                            const int64_t* cand_rows, const int* cand_lins, const int* counts,
                            int64_t r_begin, const double* miss, unsigned long long* stats,
                            long long* rec, cudaStream_t st) {
  finalize_kernel<<<1, 1, 0, st>>>(scal, win_err, win_c, cand_rows, cand_lins, counts, r_begin, miss,
                                   stats, rec);
  return cudaGetLastError();
}

__global__ void enumerate_poses_kernel(int64_t p0, int64_t np, int64_t ntrans, int64_t* rows,
                                       int* lins) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < np;
       k += (int64_t)gridDim.x * blockDim.x) {
    rows[k] = (p0 + k) / ntrans;
    lins[k] = (int)((p0 + k) % ntrans);
  }
}

cudaError_t launch_enumerate_poses(int64_t p0, int64_t np, int64_t ntrans, int64_t* rows, int* lins,
                                   cudaStream_t st) {
  if (np <= 0) return cudaSuccess;
  enumerate_poses_kernel<<<(int)std::min<int64_t>(4096, (np + 255) / 256), 256, 0, st>>>(
      p0, np, ntrans, rows, lins);
  return cudaGetLastError();
}

cudaError_t launch_rescore_compact(const double* err, int64_t ncand, double thr, int* sel,
                                   unsigned long long* nsel, cudaStream_t st,
                                   const unsigned long long* dcount,
                                   const unsigned long long* dmin, double tol) {
  if (ncand <= 0) return cudaSuccess;
  const int rb = (int)std::min<int64_t>(dcount ? 256 : 65535, (ncand + 255) / 256);
  rescore_compact_kernel<<<std::max(rb, 1), 256, 0, st>>>(err, ncand, thr, sel, nsel, dcount, dmin,
                                                          tol);
  return cudaGetLastError();
}

cudaError_t launch_exact(const ScoreParams& s, const int64_t* rows, const int* lins, const int* sel,
                         int64_t nsel, double* vals, double* out, cudaStream_t st,
                         const unsigned long long* dcount) {
  if (nsel <= 0) return cudaSuccess;
  const int nblk = (s.n + kExactThreads / 32 - 1) / (kExactThreads / 32);
  const int64_t cap_y = std::max<int64_t>(1, std::min<int64_t>(65535, 16384 / nblk));
  exact_points_kernel<<<dim3(nblk, (unsigned)std::min<int64_t>(nsel, dcount ? cap_y : 65535)),
                        kExactThreads, 0, st>>>(s, rows, lins, sel, nsel, vals, dcount);
  const int rb = (int)std::min<int64_t>(dcount ? 1024 : 65535, (nsel + 3) / 4);  // 4 warps per block
  exact_sum_kernel<<<std::max(rb, 1), 128, 0, st>>>(vals, s.n, nsel, out, dcount, s.code == kSatL0);
  return cudaGetLastError();
}

cudaError_t launch_winner(const double* err64, const int* sel, const int64_t* rows, int64_t nsel,
                          double* best_err, int64_t* best_row, int* best_c, cudaStream_t st,
                          const int* lins, const unsigned long long* dcount) {
  winner_kernel<<<1, 1024, 0, st>>>(err64, sel, rows, nsel, best_err, best_row, best_c, lins,
                                    dcount);
  return cudaGetLastError();
}

}  // namespace dses
