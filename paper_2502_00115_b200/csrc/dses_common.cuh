// dses_common.cuh -- shared device-side definitions for the B200 DSES kernels.
//
// Numerics contract:
//  * The reference bins a vote (i, j) in binary64 as
//      p  = R x_i                      ((r0*x0 + r1*x1) + r2*x2, no FMA)
//      q  = (y_j - p) * inv_bin        (_kernels.py:135-149)
//      f  = copysign(floor(|q| + 0.5), q) - lo
//    exact_bin() below reproduces that sequence with explicit __dmul_rn /
//    __dadd_rn intrinsics so nvcc cannot contract it into FMAs.
//  * The fast path bins in 32-bit fixed point (F fraction bits per bin):
//      Yq = rint(fl(y*inv_bin) * 2^F) - lo*2^F + 2^(F-1) + G     (host, exact int64)
//      Pq = rint(fl(p*inv_bin*2^F))                              (device, per rotation)
//      u  = Yq - Pq                                              (exact int32)
//    |u - (U + G) 2^F| <= 1 unit, U = (y-p)*inv_bin - lo + 1/2, so a pair whose
//    fraction lies >= G units from a bin edge is binned exactly by u >> F; the
//    rest (probability ~4G/2^F per axis) are re-binned by exact_bin().
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// DSES_DEBUG_BOUNDS: device-side bounds checks on every histogram update and
// point index (a debug build; compute-sanitizer is unavailable on the pool).
#ifdef DSES_DEBUG_BOUNDS
#include <cassert>
#define DSES_ASSERT(c) assert(c)
#else
#define DSES_ASSERT(c) ((void)0)
#endif

namespace dses {

constexpr int kTile = 32;        // points per reference group (one per lane) and per source unit
constexpr int kGuard = 2;        // guard band in fixed-point units
constexpr int kUnitCapMin = 2048;       // minimum (reference group, source unit) list capacity per round
constexpr int kDenseMaxBins = 1 << 26;  // beyond: sort-based (sparse) mode queries
// Sentinel Yq.x of empty reference slots: with |Pq| < 2^29 and W < 2^30 (or
// W = 2^31 - 1 and Pq = 0 in exact mode) u = Yq - Pq wraps to >= 2^30 > W.
constexpr int kNoRef = -3 * (1 << 29);
constexpr int kMaxComp = 16;     // dedup components up to this size stay in one warp
constexpr int kFarFlag = 1 << 12; // Yq.w: the point's dedup needs the exact path
// Yq.w bits read by the rotation-block kernel (vote_blocks_kernel):
constexpr int kPartFlag = 1 << 18;   // the point has a dedup partner
constexpr int kSplitFlag = 1 << 19;  // its component spans several groups (always exact)
constexpr int kCompOffShift = 20;    // bits 20..23: its offset from the component's first point
                                     // (components are contiguous in tile order)
constexpr int kMaxBlockRot = 32;  // rotations per block (the block kernel's R area in shared memory)
// shared-memory bytes of the rotation-matrix area (the block's rotations and
// its centre), a multiple of 16 so that the int4 areas after it stay aligned
constexpr int kRotAreaBytes = ((kMaxBlockRot + 1) * 9 * 8 + 15) / 16 * 16;
constexpr double kBlockLaneUseMax = 0.2;   // blocks when the per-rotation kernel would use fewer lanes
constexpr int kDefaultBlockShape[3] = {1, 3, 3};  // rotations per block along the Euler-index axes
#ifndef DSES_BLOCK_LIST_CAP
#define DSES_BLOCK_LIST_CAP (1 << 17)
#endif
constexpr int kBlockListCap = DSES_BLOCK_LIST_CAP;  // candidate-list entries per CTA (2 MiB of 16-byte entries)
// the list vote prefetches one segment per warp past the last: slack after the slabs
constexpr int kBlockListSlack = 32 * 32;
constexpr int kRiskBits = 10;     // fraction buckets per axis of the guard-band risk bitmaps
constexpr int kRiskWords = 3 * (1 << kRiskBits) / 32;  // words per group (3 axes)
constexpr int kVoteThreads = 1024;

enum Metric { kL2 = 0, kL1 = 1, kTruncL1 = 2, kSatL0 = 3, kTruncL2 = 4 };

struct XTile {          // spatial tile (source unit) of the (sorted) source cloud
  int start, count;
};

struct __align__(16) YTile {  // spatial tile of the (sorted) reference cloud; 3 x 16 bytes
  int lo[3];            // fixed-point bounding box of Yq over the tile
  int start;
  int hi[3];
  int count;
  int gm;               // max earlier dedup partners (lanes) of a point in the group: 0, 1, 2
  int npts;             // real reference points in the group
  int pad[2];           // pad[0]: the group has far points (no source is guard-band safe)
};
static_assert(sizeof(YTile) == 48, "YTile is loaded as three int4");

// YTile through three 16-byte read-only loads
__device__ __forceinline__ YTile load_ytile(const YTile* yt, int b) {
  const int4* q = reinterpret_cast<const int4*>(yt + b);
  const int4 a = __ldg(q), h = __ldg(q + 1), m = __ldg(q + 2);
  YTile t;
  t.lo[0] = a.x; t.lo[1] = a.y; t.lo[2] = a.z; t.start = a.w;
  t.hi[0] = h.x; t.hi[1] = h.y; t.hi[2] = h.z; t.count = h.w;
  t.gm = m.x; t.npts = m.y; t.pad[0] = m.z; t.pad[1] = 0;
  return t;
}

struct RotSource {      // where rotation r comes from
  const double* cth;    // grid tables (device), 2k+1 values; NULL -> explicit
  const double* sth;
  const double* rots;   // explicit matrices (device), r x 9
  int64_t k;
  int has_center;
  double center[9];
};

struct VoteParams {
  // lattice
  int d0, d1, d2, nbins;
  int F;                 // fraction bits; 0 => exact mode (every pair re-binned in fp64)
  unsigned fmask;        // 2^F - 1
  unsigned W0, W1, W2;   // prefilter: (unsigned)u < d*2^F + 2G
  unsigned D0, D1, D2;   // d*2^F
  double inv_bin, inv_s; // 1/bin (as the reference computes it) and inv_bin*2^F
  double flo0, flo1, flo2, fd0, fd1, fd2;
  // clouds (tile-sorted)
  int n, m, nxt, nyt;
  int m_pad;             // reference slots (yq / ys / near lists are m_pad long)
  int unit_cap;          // capacity of the per-round (group, unit) list in shared memory
  const double* xs;      // (n,3) f64, X tile order
  const double* ys;      // (m,3) f64, Y tile order
  const int4* yq;        // (m) fixed-point Yq in group order; w = lanes+1 of up to two earlier
                         // dedup partners (bits 0-5, 6-11) or kFarFlag (exact path)
  const int* near_off;   // (m+1) CSR offsets of the full dedup near lists (tile order)
  const int* near_idx;   // near neighbours j' < j with |y_j - y_j'|_inf < bin (1+1e-6)
  const XTile* xt;       // source units of <= kTile points
  const YTile* yt;       // reference groups of <= kTile points
  unsigned gthr;         // a pair whose min fraction over the axes is < gthr is re-binned exactly
  const unsigned* risk;  // per group kRiskWords: guard-band risk bitmaps (dses_capi.cu)
  int risk_shift;        // F - kRiskBits (bucket of a fraction); 0 with every group unsafe
  RotSource rot;
  int64_t r_begin, r_count;
  // outputs (indexed r - r_begin)
  int* counts;
  int* lins;
  int* ties;
  unsigned long long* stats;  // [pairs, votes, rechecks, rotation counter (zeroed per launch)]
  // global fallbacks when the histogram / rotated points do not fit shared memory
  unsigned* hist_global;      // per-CTA slabs of hist_words (u32 counts when !count16)
  int4* p_global;             // per-CTA slabs of n_pad entries
  int hist_words;             // u32 words per histogram (padded to a multiple of 4)
  int n_pad;
  int count16;                // two 16-bit counts per word (n < 65536)
  // rotation blocks (vote_blocks_kernel): boxes of up to blk_s[0] x blk_s[1]
  // x blk_s[2] neighbouring grid rotations share one candidate-pair list
  // built at the block's centre rotation with each source unit's window
  // widened by its points' maximal motion over the block
  int blk_s[3];               // sides along the three Euler-index axes (0: per-rotation kernel)
  int jbits;                  // entry word = i << (jbits + 4) | j << 4 | c; j = m_pad: the empty sentinel
  int ishift;                 // jbits + 4: the source index's place in a 16-byte entry's .w
  int list_cap;               // entries per CTA slab (multiple of 32)
  unsigned* list;             // per-CTA slabs
  long long* redo;            // rotations of blocks whose list overflowed ...
  unsigned long long* redo_n; // ... and their number: vote_kernel runs them (redo mode)
};

struct ScoreParams {     // scoring kernels (dses_score.cu)
  int n, m;
  const double* x;        // (n,3) source, ORIGINAL order (the serial sum order)
  const double* ys0;      // reference columns sorted by axis 0 (engines.py:133-140)
  const double* ys1;
  const double* ys2;
  const float4* ysf;      // same order, fp32 (screen)
  RotSource rot;
  double bin_size;
  int64_t ilo0, ilo1, ilo2;
  int d1, d2;
  int code;
  double param;
  float paramf, halff;    // fp32 metric parameter and sat_l0 half width
  float amb;              // sat_l0 fp32 ambiguity margin (absolute)
  const double* tvec;     // explicit translations (row-indexed) instead of decoding bins
  int exh_k;              // >= 0: exhaustive-search translations t = tcen + (f - exh_k) * bin
  double tcen[3];         //       (engines.py:168-169), f = the lattice index of lin
  // uniform grid over the reference cloud (screen nearest-neighbour search)
  const int2* gcell;      // per cell: [begin, end) into gpts
  const float4* gpts;     // reference points sorted by cell (fp32; .w = int index in axis-0 order)
  float gorg[3];          // grid origin
  float gh, ginv;         // cell size and 1/cell size
  int gdim[3];            // cells per axis
  float gppc;             // reference points per non-empty cell (exact re-score: grid vs window)
};

struct SparseParams {    // sort-based mode queries (dses_sparse.cu)
  int n, m;
  const double* x;        // (n, 3) source (any order: keys carry i)
  const double* y;        // (m, 3) reference
  double inv_bin;
  double flo0, flo1, flo2, fd0, fd1, fd2;
  int64_t d1, d2;
  RotSource rot;
};

// ---------------------------------------------------------------------------
// exact binary64 helpers (no contraction)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// p_k = (r_k0*x0 + r_k1*x1) + r_k2*x2  (_kernels.py:135-137, 320-322 without t)
__device__ __forceinline__ double rot_row(const double* R, int k, double x0, double x1, double x2) {
  return dadd(dadd(dmul(R[3 * k], x0), dmul(R[3 * k + 1], x1)), dmul(R[3 * k + 2], x2));
}

// Grid entry e (row-major) of Rz(xi) Ry(phi) Rx(theta) for angle indices (a,b,c),
// in numpy's evaluation order (geometry.py:279-287).
__device__ __forceinline__ double grid_entry(const double* cth, const double* sth, int64_t a,
                                             int64_t b, int64_t c, int e) {
  const double c1 = cth[a], s1 = sth[a], c2 = cth[b], s2 = sth[b], c3 = cth[c], s3 = sth[c];
  switch (e) {
    case 0: return dmul(c3, c2);
    case 1: return dadd(dmul(-s3, c1), dmul(dmul(c3, s2), s1));
    case 2: return dadd(dmul(s3, s1), dmul(dmul(c3, s2), c1));
    case 3: return dmul(s3, c2);
    case 4: return dadd(dmul(c3, c1), dmul(dmul(s3, s2), s1));
    case 5: return dadd(dmul(-c3, s1), dmul(dmul(s3, s2), c1));
    case 6: return -s2;
    case 7: return dmul(c2, s1);
    default: return dmul(c2, c1);
  }
}

// Entry e of rotation r: grid (optionally centre-multiplied, engines.py:122-126,
// summation ((C a0 G 0c + C a1 G 1c) + C a2 G 2c)) or explicit.
__device__ __forceinline__ double rotation_entry(const RotSource& rs, int64_t r, int e) {
  if (rs.rots) return rs.rots[9 * r + e];
  const int64_t n = 2 * rs.k + 1;
  const int64_t a = r / (n * n), b = (r / n) % n, c = r % n;
  if (!rs.has_center) return grid_entry(rs.cth, rs.sth, a, b, c, e);
  const int row = e / 3, col = e % 3;
  const double g0 = grid_entry(rs.cth, rs.sth, a, b, c, col);
  const double g1 = grid_entry(rs.cth, rs.sth, a, b, c, 3 + col);
  const double g2 = grid_entry(rs.cth, rs.sth, a, b, c, 6 + col);
  return dadd(dadd(dmul(rs.center[3 * row], g0), dmul(rs.center[3 * row + 1], g1)),
              dmul(rs.center[3 * row + 2], g2));
}

// Reference binning of one pair, _kernels.py:144-152.  Returns true when the
// vote lands inside the window; *lin gets the flat bin (f0*d1 + f1)*d2 + f2.
__device__ __forceinline__ bool exact_bin(const VoteParams& p, double p0, double p1, double p2,
                                          const double* yj, int* lin) {
  const double q0 = dmul(dsub(yj[0], p0), p.inv_bin);
  const double f0 = dsub(copysign(floor(dadd(fabs(q0), 0.5)), q0), p.flo0);
  const double q1 = dmul(dsub(yj[1], p1), p.inv_bin);
  const double f1 = dsub(copysign(floor(dadd(fabs(q1), 0.5)), q1), p.flo1);
  const double q2 = dmul(dsub(yj[2], p2), p.inv_bin);
  const double f2 = dsub(copysign(floor(dadd(fabs(q2), 0.5)), q2), p.flo2);
  const bool ok = (f0 >= 0.0) & (f0 < p.fd0) & (f1 >= 0.0) & (f1 < p.fd1) & (f2 >= 0.0) &
                  (f2 < p.fd2);
  if (ok) *lin = (int)dadd(dmul(dadd(dmul(f0, p.fd1), f1), p.fd2), f2);
  return ok;
}

// Combine (best, lin, ties) triples: higher count wins, equal counts keep the
// smaller flat bin and add their tie counts (_kernels.py:159-170).
__device__ __forceinline__ void mode_combine(int& best, int& lin, int& ties, int ob, int ol, int ot) {
  if (ob > best) { best = ob; lin = ol; ties = ot; }
  else if (ob == best) { lin = min(lin, ol); ties += ot; }
}

}  // namespace dses
