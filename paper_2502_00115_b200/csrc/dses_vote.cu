// dses_vote.cu -- phase 1 of DSES on B200: rotate, vote, take the histogram mode.
//
// Replaces _kernels.mode_dense_batch / _mode_dense_one (_kernels.py:109-193)
// and mode_sparse_batch (_kernels.py:196-294): per rotation r, every pair
// (source i, reference j) votes for translation bin round((y_j - R x_i)/bin)
// inside the window [lo, lo+d); a bin's count is the number of DISTINCT source
// points voting for it; the result is (max count, smallest flat bin at the max,
// number of bins at the max).
//
// B200 design:
//  * persistent CTAs (one per SM when the histogram lives in shared memory),
//    each looping over rotations; the rotation matrix is generated in-kernel
//    from the per-axis trig tables (nothing is materialised in HBM);
//  * the histogram is 16-bit counts packed two per word in shared memory
//    (41^3 bins -> 135 KB) updated with shared atomics (~8 per clock per SM
//    measured); the scan that extracts the mode also re-zeroes it;
//  * both clouds are pre-sorted into 32-point spatial tiles; a (source tile,
//    reference tile) pair is skipped when the rotated source tile's bounding
//    sphere cannot produce an in-window vote -- one lane-parallel test per 32
//    tile pairs, ballot, then only surviving tile pairs are swept;
//  * the sweep keeps one reference point per lane in registers and
//    broadcasts rotated source points from shared memory: 3 IADD + 3 ISETP per
//    pair in 32-bit fixed point (exact integer subtraction); pairs within
//    kGuard units of a bin edge are re-binned in exact binary64;
//  * per-source dedup (a bin counts each source once, _kernels.py:153-158)
//    without a last[] array: a vote (i, j) is dropped iff some j' < j from
//    j's precomputed near list (|y_j - y_j'|_inf < bin) lands in the same bin
//    for the same i.  Two reference points can only share a bin if they are
//    closer than one bin per axis, so the rule is exact and order-free.
#include <climits>
#include <cstdio>
#include <mutex>
#include "dses_common.cuh"

namespace dses {

// Fast fixed-point bin of pair (Yq, Pq); returns 0 = out of window, 1 = in
// window (lin set), 2 = within the guard band (caller re-bins exactly).
__device__ __forceinline__ int fast_bin(const VoteParams& p, int u0, int u1, int u2, int* lin) {
  const unsigned g2 = 2u * kGuard;
  const bool near = (((unsigned)u0 & p.fmask) < g2) | (((unsigned)u1 & p.fmask) < g2) |
                    (((unsigned)u2 & p.fmask) < g2);
  if (near) return 2;
  const bool in = ((unsigned)u0 < p.D0) & ((unsigned)u1 < p.D1) & ((unsigned)u2 < p.D2);
  if (!in) return 0;
  *lin = ((u0 >> p.F) * p.d1 + (u1 >> p.F)) * p.d2 + (u2 >> p.F);
  return 1;
}

// Full bin decision for pair (i, j): fast path, exact fallback.
__device__ __forceinline__ bool pair_bin(const VoteParams& p, const double* R, const int4& P,
                                         int i, const int4& Y, int j, int* lin, unsigned& rechecks) {
  const int s = fast_bin(p, Y.x - P.x, Y.y - P.y, Y.z - P.z, lin);
  if (s != 2) return s == 1;
  ++rechecks;
  const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
  const double p0 = rot_row(R, 0, x0, x1, x2);
  const double p1 = rot_row(R, 1, x0, x1, x2);
  const double p2 = rot_row(R, 2, x0, x1, x2);
  return exact_bin(p, p0, p1, p2, p.ys + 3 * j, lin);
}

constexpr int kRare = 64;       // per-warp list of deferred (i, j) pairs

// Can a source box [lo, hi] and the reference tile bbox produce u = Yq - Pq in [0, W)?
__device__ __forceinline__ bool boxes_meet(const VoteParams& p, const YTile& yt, const int4& lo,
                                           const int4& hi) {
  return (yt.hi[0] - lo.x >= 0) & (yt.lo[0] - hi.x < (int)p.W0) & (yt.hi[1] - lo.y >= 0) &
         (yt.lo[1] - hi.y < (int)p.W1) & (yt.hi[2] - lo.z >= 0) & (yt.lo[2] - hi.z < (int)p.W2);
}

// Lane index and lower-lanes mask from the special registers (one S2R each
// wherever the compiler re-materialises them).
__device__ __forceinline__ unsigned lane_sr() {
  unsigned r;
  asm("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned lanemask_lt_sr() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// 32-bit shared-memory accessors (shared window addresses computed once).
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void reds_add(uint32_t a, unsigned v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t a, const int4& v) {
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t a, int x, int y) {
  asm volatile("st.shared.v2.s32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ int2 lds_v2(uint32_t a) {
  int2 v;
  asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

template <bool HSMEM>
__device__ __forceinline__ void hist_inc(unsigned* hist, uint32_t hist_sh, int lin) {
  if (HSMEM) reds_add(hist_sh + 2u * (unsigned)(lin & ~1), (lin & 1) ? 0x10000u : 1u);
  else atomicAdd(&hist[lin], 1u);
}

// The exact general path for one deferred pair (i, j): reference binning
// (fast fixed point, binary64 in the guard band) and the full near list of j
// (every j' < j with |y_j - y_j'|_inf < bin): the vote counts unless some j'
// lands in the same bin for the same i (_kernels.py:144-158).
// Returns (votes << 16) | rechecks.
template <bool HSMEM, bool PSMEM>
__device__ __forceinline__ unsigned vote_exact(const VoteParams& p, const double* R, const int4* P,
                                            unsigned* hist, uint32_t hist_sh, int i, int j) {
  unsigned rechecks = 0;
  const int4 Pi = PSMEM ? P[i] : __ldcg(&P[i]);
  int lin;
  if (!pair_bin(p, R, Pi, i, p.yq[j], j, &lin, rechecks)) return rechecks;
  const int e1 = p.near_off[j + 1];
  for (int k = p.near_off[j]; k < e1; ++k) {
    const int jj = p.near_idx[k];
    int lin2;
    if (pair_bin(p, R, Pi, i, p.yq[jj], jj, &lin2, rechecks) && lin2 == lin) return rechecks;
  }
  DSES_ASSERT(lin >= 0 && lin < p.nbins && i >= 0 && i < p.n && j >= 0 && j < p.m_pad);
  hist_inc<HSMEM>(hist, hist_sh, lin);
  return (1u << 16) | rechecks;
}

// Flush a warp's deferred list (n entries, <= kRare) through vote_exact.
// Inlined, with a warp-uniform trip count: ptxas then proves the warp
// converged around the slot loop's shuffles / votes (a call into a
// non-inlined divergent function made it guard each of them with BRA.DIV).
template <bool HSMEM, bool PSMEM>
__device__ __forceinline__ unsigned flush_rare(const VoteParams& p, const double* R,
                                                 const int4* P, unsigned* hist, uint32_t hist_sh,
                                                 uint32_t rare_sh, int n, int lane) {
  unsigned acc = 0;
  __syncwarp();
  for (int base = 0; base < n; base += 32) {
    const int e = base + lane;
    if (e < n) {
      const int2 ij = lds_v2(rare_sh + 8u * (unsigned)e);
      acc += vote_exact<HSMEM, PSMEM>(p, R, P, hist, hist_sh, ij.x, ij.y);
    }
  }
  __syncwarp();
  return acc;
}

// Predicated shared-memory reduction.
__device__ __forceinline__ void reds_add_if(uint32_t a, unsigned v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}"
               ::"r"(a), "r"(v), "r"((unsigned)pred) : "memory");
}


struct Lane {          // per-warp deferred list state (warp-uniform)
  uint32_t rare_sh;
  int nrare;
  unsigned rechecks;
};

// Generic pointers of the exact path, published once per CTA: the slot loop
// reads them only when it flushes (otherwise the compiler re-derives them
// from kernel parameters in every slot).
__shared__ const double* g_exR;
__shared__ const int4* g_exP;
__shared__ unsigned* g_exH;
__shared__ unsigned g_dummy[32];   // per-lane sink of non-voting unconditional atomics
#define g_dummy_sh ((uint32_t)__cvta_generic_to_shared(g_dummy))

// Append the lanes in `dm` (pairs (i, j)) to the warp's exact-path list.
template <bool HSMEM, bool PSMEM>
__device__ __forceinline__ void defer_pairs(const VoteParams& p, uint32_t hist_sh, Lane& L,
                                            unsigned dm, bool mine, int i, int j, int lane,
                                            unsigned lanemask_lt) {
  if (mine) sts_v2(L.rare_sh + 8u * (unsigned)(L.nrare + __popc(dm & lanemask_lt)), i, j);
  L.nrare += __popc(dm);
  if (L.nrare > kRare - 32) {
    L.rechecks += flush_rare<HSMEM, PSMEM>(p, g_exR, g_exP, g_exH, hist_sh, L.rare_sh, L.nrare,
                                           lane) & 0xffffu;
    L.nrare = 0;
  }
}

// Fast-path constants in per-lane registers.
struct FastK {
  unsigned W0, W1, W2, fmask, gthr, d1, d2;
  int F;
  unsigned negP;  // -(2^F): fraction = u + (u >> F) * negP on the multiply pipe
};

// Fixed-point decision for one pair: candidate (inside the guard-extended
// window), near (within the guard band of a bin edge: exact path) and bin.
struct PairBin {
  bool cand, near;
  unsigned lin;
};
__device__ __forceinline__ PairBin fixed_bin(const FastK& k, const int4& Y, const int4& Pi) {
  PairBin r;
  const unsigned u0 = (unsigned)(Y.x - Pi.x), u1 = (unsigned)(Y.y - Pi.y), u2 = (unsigned)(Y.z - Pi.z);
  r.cand = (u0 < k.W0) & (u1 < k.W1) & (u2 < k.W2);
  // a candidate with every fraction >= 2G lies inside [0, D) (u in [D, W) has
  // a fraction < 2G) and its fixed-point bin u >> F is the exact bin
  // the bins u >> F are needed anyway; the fractions u - (u >> F) * 2^F then
  // cost one IMAD each (FMA pipe) instead of an AND on the saturated ALU pipe
  const unsigned q0 = u0 >> k.F, q1 = u1 >> k.F, q2 = u2 >> k.F;
  r.near = r.cand & (__vimin3_u32(u0 + q0 * k.negP, u1 + q1 * k.negP, u2 + q2 * k.negP) < k.gthr);
  r.lin = (q0 * k.d1 + q1) * k.d2 + q2;
  return r;
}

// The same for a guard-band-safe (source, group) pair (risk bitmaps,
// dses_capi.cu): no fraction can be near a bin edge, so the near test is
// skipped; every candidate is decided.
__device__ __forceinline__ PairBin fixed_bin_safe(const FastK& k, const int4& Y, const int4& Pi) {
  PairBin r;
  const unsigned u0 = (unsigned)(Y.x - Pi.x), u1 = (unsigned)(Y.y - Pi.y), u2 = (unsigned)(Y.z - Pi.z);
  r.cand = (u0 < k.W0) & (u1 < k.W1) & (u2 < k.W2);
  r.near = false;
  r.lin = ((u0 >> k.F) * k.d1 + (u1 >> k.F)) * k.d2 + (u2 >> k.F);
  return r;
}

template <bool HSMEM>
__device__ __forceinline__ void vote_if(unsigned* hist, uint32_t hist_sh, unsigned lin, bool ok,
                                        unsigned nbins = 0xffffffffu) {
  DSES_ASSERT(!ok || lin < nbins);
  // 1 << 16*(lin & 1) as a wrapping funnel shift of lin*16 (the multiply is
  // on the FMA pipe): one ALU instruction instead of an AND and a shift
  if (HSMEM) reds_add_if(hist_sh + ((lin + lin) & ~3u), __funnelshift_l(0u, 1u, lin << 4), ok);
  else if (ok) atomicAdd(&hist[lin], 1u);
}

// Source point i (broadcast) against the warp's reference group (lane = one
// reference point j, registers).  A lane votes for its fixed-point bin when
// the pair is decided (a candidate outside the guard band) and no earlier
// dedup partner of j -- a lane of the same group, its key arrives by
// shuffle -- is decided in the same bin (_kernels.py:153-158: a bin counts
// each source once).  Pairs in the guard band, pairs whose partner is in the
// guard band, and "far" points take the exact path.  GP = number of partner
// shuffles the group needs (0, 1, 2).
template <bool HSMEM, bool PSMEM, int GP, int NS, bool SAFE>
__device__ __forceinline__ void vote_slot(const VoteParams& p, const FastK& fk, const double* R,
                                          const int4* P, unsigned* hist, uint32_t hist_sh, Lane& L,
                                          const int4& Y, int l0, int l1, uint32_t src_sh, int j,
                                          int lane, unsigned lanemask_lt) {
  // NS source points per call: their independent work interleaves and the
  // warp votes / loop overhead are shared.
  PairBin b[NS];
  int is[NS];
  bool any = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    // the unit's surviving sources, staged (Pq, i) per warp: uniform address
    const int4 Pi = lds_v4(src_sh + 16u * (unsigned)s);
    is[s] = Pi.w;
    b[s] = SAFE ? fixed_bin_safe(fk, Y, Pi) : fixed_bin(fk, Y, Pi);
    any |= b[s].cand;
  }
  if (!__any_sync(0xffffffffu, any)) return;
  bool anynear = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) anynear |= b[s].near;
  if (SAFE || !__any_sync(0xffffffffu, anynear)) {
    // common case: no candidate of the slot is near a bin edge, so every
    // candidate is decided and a partner's key is its exact bin or -1
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      bool ok = b[s].cand;
      if (GP > 0) {
        const int key = b[s].cand ? (int)b[s].lin : -1;
        ok &= __shfl_sync(0xffffffffu, key, l0 & 31) != key;
        if (GP > 1) ok &= __shfl_sync(0xffffffffu, key, l1 & 31) != key;
      }
      if (HSMEM) {
        // unconditional: a lane that does not vote adds to its own dummy word
        // (conflict-free), so no branch / reconvergence around the atomic
        const unsigned lin = b[s].lin;
        const uint32_t a = ok ? hist_sh + ((lin + lin) & ~3u) : g_dummy_sh + 4u * (unsigned)lane;
        reds_add(a, __funnelshift_l(0u, 1u, lin << 4));
      } else
        vote_if<HSMEM>(hist, hist_sh, b[s].lin, ok, (unsigned)p.nbins);
    }
    return;
  }
  bool defer[NS], anydef = false;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const bool decided = b[s].cand & !b[s].near;
    bool ok = decided;
    defer[s] = b[s].near;
    if (GP > 0) {
      const int key = decided ? (int)b[s].lin : (b[s].near ? -2 : -1);
      const int k0 = __shfl_sync(0xffffffffu, key, l0 & 31);
      bool dup = k0 == key;  // l0 is always a lane: a partner or a safe one
      bool und = k0 == -2;
      if (GP > 1) {
        const int k1 = __shfl_sync(0xffffffffu, key, l1 & 31);
        dup |= k1 == key;
        und |= k1 == -2;
      }
      dup &= decided;
      ok = decided & !dup & !und;
      defer[s] = b[s].near | (decided & !dup & und);
    }
    vote_if<HSMEM>(hist, hist_sh, b[s].lin, ok, (unsigned)p.nbins);
    DSES_ASSERT(is[s] >= 0 && is[s] < p.n && j >= 0 && j < p.m_pad);
    anydef |= defer[s];
  }
  if (__any_sync(0xffffffffu, anydef)) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const unsigned dm = __ballot_sync(0xffffffffu, defer[s]);
      if (dm) defer_pairs<HSMEM, PSMEM>(p, hist_sh, L, dm, defer[s], is[s], j, lane, lanemask_lt);
    }
  }
}

// RISK: guard-band risk bitmaps in use (small reference clouds; dses_capi.cu)
// REDO: the rotations come from a device-side list (redo / redo_n): those of
// rotation blocks whose candidate list overflowed (vote_blocks_kernel)
template <bool HSMEM, bool PSMEM, bool RISK, bool REDO = false>
__global__ void __launch_bounds__(kVoteThreads, 1) vote_kernel(const VoteParams p) {
  if (REDO && *p.redo_n == 0) return;  // (the usual case: no block overflowed)
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nthreads = blockDim.x, nwarps = nthreads >> 5, warp = tid >> 5;

  size_t off = 0;
  unsigned* hist;
  if (HSMEM) { hist = reinterpret_cast<unsigned*>(smem); off += (size_t)p.hist_words * 4; }
  else hist = p.hist_global + (size_t)blockIdx.x * p.hist_words;
  int4* P;
  if (PSMEM) { P = reinterpret_cast<int4*>(smem + off); off += (size_t)p.n_pad * 16; }
  else P = p.p_global + (size_t)blockIdx.x * p.n_pad;
  const int nxc = (p.nxt + 31) >> 5;                // chunks of 32 units
  int4* XB = reinterpret_cast<int4*>(smem + off);  // [2*nxt] rotated unit boxes (lo, hi)
  int4* CB = XB + 2 * p.nxt;                       // [2*nxc] their union per chunk
  off += (size_t)(p.nxt + nxc) * 32;
  double* R = reinterpret_cast<double*>(smem + off);
  off += kRotAreaBytes;                            // (the block kernel's layout: same offsets)
  int* red = reinterpret_cast<int*>(smem + off);    // [3 * 32] reduction scratch + counters
  off += 4 * 32 * 4;
  unsigned* units = reinterpret_cast<unsigned*>(smem + off);  // [unit_cap] (group << 16 | unit)
  off += (size_t)p.unit_cap * 4;
  int2* rare = reinterpret_cast<int2*>(smem + off) + warp * kRare;
  off += (size_t)nwarps * kRare * 8;
  int4* stage = reinterpret_cast<int4*>(smem + off) + warp * 32;  // a unit's surviving sources
  const uint32_t stage_sh = (uint32_t)__cvta_generic_to_shared(stage);

  int* s_nunits = red + 96;
  int* s_next = red + 97;
  int* s_ovf = red + 98;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  const uint32_t P_sh = PSMEM ? (uint32_t)__cvta_generic_to_shared(P) : 0u;
  // fast-path constants through shared memory: loaded into regular registers
  // once, instead of being re-loaded into uniform registers in the hot loop
  __shared__ __align__(16) unsigned kc[12];
  __shared__ unsigned s_pairs[kVoteThreads / 32];  // per-warp evaluated pairs of this rotation
  if (tid == 0) {
    kc[0] = p.W0; kc[1] = p.W1; kc[2] = p.W2; kc[3] = p.fmask; kc[4] = p.gthr;
    kc[5] = (unsigned)p.d1; kc[6] = (unsigned)p.d2; kc[7] = (unsigned)p.F;
    kc[8] = HSMEM ? (uint32_t)__cvta_generic_to_shared(hist) : 0u;
    kc[9] = 0u - (1u << p.F);
    kc[10] = kc[11] = 0u;
    g_exR = R;
    g_exP = P;
    g_exH = hist;
  }
  __syncthreads();
  const uint32_t hist_sh = kc[8];
  if (lane == 0) s_pairs[warp] = 0;
  unsigned long long st_pairs = 0;
  Lane L;
  // opaque copy: a register, not re-derived from kernel parameters per slot
  asm volatile("mov.u32 %0, %1;" : "=r"(L.rare_sh) : "r"((uint32_t)__cvta_generic_to_shared(rare)));
  L.nrare = 0;
  L.rechecks = 0;

  uint4* hist4 = reinterpret_cast<uint4*>(hist);
  const int nw4 = p.hist_words >> 2;
  for (int w = tid; w < nw4; w += nthreads) {
    if (HSMEM) hist4[w] = make_uint4(0, 0, 0, 0); else __stcg(&hist4[w], make_uint4(0, 0, 0, 0));
  }

  unsigned long long st_votes = 0;
  const bool exact_mode = (p.F == 0);
  // Rounds: each tries up to `gmax` reference groups (their chunk masks live
  // at the tail of `units`, the rest holds the round's surviving (group,
  // unit) pairs); a round whose pairs overflow the list keeps the groups
  // below the first one that overflowed and the next round restarts there
  // (a one-group round when even the first group overflowed: its <= nxt
  // units always fit).  With typical overlap a rotation is one round.
  // (the RISK specialisation -- small reference clouds -- keeps worst-case
  // sized rounds: no overflow bookkeeping on its hot path)
  constexpr bool OVF = !RISK;
  const int gmax = OVF ? max(1, min(min(p.nyt, p.unit_cap / 4), p.unit_cap - p.nxt - 1))
                       : max(1, p.unit_cap / max(1, p.nxt + 1));
  const bool masks = !exact_mode && nxc > 1 && nxc <= 32;

  // rotations: the first one static, the rest from a global queue (the cost
  // of a rotation varies with its angle; dynamic claims balance the tail)
  __shared__ long long s_rr;
  const int64_t r_count = REDO ? (int64_t)*p.redo_n : p.r_count;
  for (int64_t rr = blockIdx.x; rr < r_count;) {
    const int64_t r = REDO ? p.redo[rr] : p.r_begin + rr;
    if (tid < 9) R[tid] = rotation_entry(p.rot, r, tid);
    __syncthreads();

    // ---- A: rotated source points in fixed point (binary64 in the reference's
    //      operation order, then one rounding); warp = source unit, lane =
    //      point, and the unit's exact rotated bounding box (fixed point, the
    //      same values the per-source test sees) by warp min/max reductions --
    //      much tighter than a rotated bounding sphere for flat units
    for (int a = warp; a < p.nxt; a += nwarps) {
      const int2 U = __ldg(reinterpret_cast<const int2*>(p.xt + a));  // start, count
      const bool valid = lane < U.y;
      const int i = U.x + (valid ? lane : 0);
      int4 v = make_int4(0, 0, 0, 0);
      if (valid && !exact_mode) {
        const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
        v.x = __double2int_rn(dmul(rot_row(R, 0, x0, x1, x2), p.inv_s));
        v.y = __double2int_rn(dmul(rot_row(R, 1, x0, x1, x2), p.inv_s));
        v.z = __double2int_rn(dmul(rot_row(R, 2, x0, x1, x2), p.inv_s));
      }
      if (valid) { if (PSMEM) P[i] = v; else __stcg(&P[i], v); }
      int4 lo, hi;
      if (exact_mode) {
        lo = make_int4(INT_MIN / 4, INT_MIN / 4, INT_MIN / 4, U.x);
        hi = make_int4(INT_MAX / 4, INT_MAX / 4, INT_MAX / 4, U.x + U.y);
      } else {
        lo = make_int4(__reduce_min_sync(0xffffffffu, valid ? v.x : INT_MAX),
                       __reduce_min_sync(0xffffffffu, valid ? v.y : INT_MAX),
                       __reduce_min_sync(0xffffffffu, valid ? v.z : INT_MAX), U.x);
        hi = make_int4(__reduce_max_sync(0xffffffffu, valid ? v.x : INT_MIN),
                       __reduce_max_sync(0xffffffffu, valid ? v.y : INT_MIN),
                       __reduce_max_sync(0xffffffffu, valid ? v.z : INT_MIN), U.x + U.y);
      }
      if (lane == 0) { XB[2 * a] = lo; XB[2 * a + 1] = hi; }
    }
    __syncthreads();
    for (int c = warp; c < nxc; c += nwarps) {  // warp = chunk, lane = unit: chunk union boxes
      const int t = 32 * c + lane;
      const bool valid = t < p.nxt;
      int4 lo = valid ? XB[2 * t] : make_int4(INT_MAX, INT_MAX, INT_MAX, 0);
      int4 hi = valid ? XB[2 * t + 1] : make_int4(INT_MIN, INT_MIN, INT_MIN, 0);
      lo.x = __reduce_min_sync(0xffffffffu, lo.x);
      lo.y = __reduce_min_sync(0xffffffffu, lo.y);
      lo.z = __reduce_min_sync(0xffffffffu, lo.z);
      hi.x = __reduce_max_sync(0xffffffffu, hi.x);
      hi.y = __reduce_max_sync(0xffffffffu, hi.y);
      hi.z = __reduce_max_sync(0xffffffffu, hi.z);
      if (lane == 0) { CB[2 * c] = lo; CB[2 * c + 1] = hi; }
    }
    __syncthreads();

    // ---- B: votes, in rounds over reference groups [b0, b1).
    //  B1  warp w tests groups b0+w, b0+w+nwarps, ... against every source
    //      unit (one per lane); overlapping (group, unit) pairs are compacted
    //      into `units` as b << 16 | a;
    //  B2  warps take units dynamically: lane = one reference point, or one
    //      dedup component of up to four points, in registers; each lane
    //      tests one source point of the unit against the group's box, then
    //      every surviving source i is broadcast from shared memory and voted
    //      in place (slot_single / slot_multi).
    // Rounds of up to gmax groups.  OVF: a round whose (group, unit) pairs
    // overflowed the list keeps the groups below its first overflowing group
    // and the next round restarts there (a one-group round when that was its
    // first group: its <= nxt units always fit).
    for (int b0 = 0, gnext = gmax; b0 < p.nyt;) {
      const int b1 = min(p.nyt, b0 + (OVF ? gnext : gmax));
      if (tid == 0) { *s_nunits = 0; *s_next = 0; if (OVF) *s_ovf = b1; }
      // which 32-unit chunks each group can reach: one thread per group
      // (instead of a warp-uniform test per (group, chunk))
      const int cap_u = p.unit_cap - gmax;  // unit-list capacity of the round
      unsigned* gmask = reinterpret_cast<unsigned*>(units) + cap_u;
      if (masks)
        for (int k = tid; k < b1 - b0; k += nthreads) {
          const YTile yg = load_ytile(p.yt, b0 + k);
          unsigned mk = 0;
          for (int c = 0; c < nxc; ++c)
            if (boxes_meet(p, yg, CB[2 * c], CB[2 * c + 1])) mk |= 1u << c;
          gmask[k] = mk;
        }
      __syncthreads();
      for (int b = b0 + warp; b < b1; b += nwarps) {
        const YTile yt = load_ytile(p.yt, b);
        if (masks) {
          for (unsigned mk = gmask[b - b0]; mk; mk &= mk - 1) {
            const int a = 32 * (__ffs(mk) - 1) + lane;
            const bool ov = a < p.nxt && boxes_meet(p, yt, XB[2 * a], XB[2 * a + 1]);
            const unsigned m = __ballot_sync(0xffffffffu, ov);
            if (m) {
              int slot = 0;
              if (lane == 0) {
                slot = atomicAdd(s_nunits, __popc(m));
                if (OVF && slot + __popc(m) > cap_u) atomicMin(s_ovf, b);
              }
              slot = __shfl_sync(0xffffffffu, slot, 0);
              if (OVF) {
                slot += __popc(m & lanemask_lt);
                if (ov && slot < cap_u) units[slot] = ((unsigned)b << 16) | (unsigned)a;
              } else if (ov) {
                units[slot + __popc(m & lanemask_lt)] = ((unsigned)b << 16) | (unsigned)a;
              }
            }
          }
          continue;
        }
        for (int a0 = 0; a0 < p.nxt; a0 += 32) {
          // whole chunk outside the group's reach: one warp-uniform test
          if (nxc > 1 && !exact_mode &&
              !boxes_meet(p, yt, CB[2 * (a0 >> 5)], CB[2 * (a0 >> 5) + 1]))
            continue;
          const int a = a0 + lane;
          const bool ov = a < p.nxt && (exact_mode || boxes_meet(p, yt, XB[2 * a], XB[2 * a + 1]));
          const unsigned m = __ballot_sync(0xffffffffu, ov);
          if (m) {
            int slot = 0;
            if (lane == 0) {
              slot = atomicAdd(s_nunits, __popc(m));
              if (OVF && slot + __popc(m) > cap_u) atomicMin(s_ovf, b);
            }
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (OVF) {
              slot += __popc(m & lanemask_lt);
              if (ov && slot < cap_u) units[slot] = ((unsigned)b << 16) | (unsigned)a;
            } else if (ov) {
              units[slot + __popc(m & lanemask_lt)] = ((unsigned)b << 16) | (unsigned)a;
            }
          }
        }
      }
      __syncthreads();
      const int nunits = OVF ? min(*s_nunits, cap_u) : *s_nunits;
      const unsigned ovf = OVF ? (unsigned)*s_ovf : 0xffffffffu;  // groups >= ovf: next round
      // sparse overlap (< 1/4 of the round's (group, unit) pairs) means light
      // units: claim three at a time to amortise the claim; dense overlap
      // (heavy units) claims one at a time to keep the round's tail balanced
      const int kpop = (4 * (int64_t)nunits < (int64_t)(b1 - b0) * p.nxt) ? 3 : 1;
      for (int u = nunits, uend = nunits;; ++u) {
        if (u >= uend) {  // claim the next kpop units
          if (lane == 0) u = atomicAdd(s_next, kpop);
          u = __shfl_sync(0xffffffffu, u, 0);
          if (u >= nunits) break;
          uend = min(nunits, u + kpop);
        }
        const unsigned unit = units[u];
        if (OVF && (unit >> 16) >= ovf) continue;  // warp-uniform
        const YTile yt = load_ytile(p.yt, (int)(unit >> 16));
        const int2 U = __ldg(reinterpret_cast<const int2*>(p.xt + (unit & 0xffffu)));
        const int ustart = U.x, ucount = U.y;
        const int gp = yt.gm;  // partner shuffles this group needs (warp-uniform)
        const bool valid = lane < yt.count;
        const int j = yt.start + (valid ? lane : 0);
        int4 Y = __ldg(&p.yq[j]);
        if (!valid) Y = make_int4(kNoRef, 0, 0, 0);
        // far lanes carry an all-ones guard threshold: every candidate of
        // theirs is "near" (exact path)
        // the fast-path constants come from shared memory per unit (nothing of
        // them stays live in registers outside the slot loop)
        FastK fkl;
        {
          const uint4 k0 = *reinterpret_cast<const uint4*>(kc);
          const uint4 k1 = *reinterpret_cast<const uint4*>(kc + 4);
          fkl.W0 = k0.x; fkl.W1 = k0.y; fkl.W2 = k0.z; fkl.fmask = k0.w;
          fkl.gthr = (Y.w & kFarFlag) ? 0xffffffffu : k1.x;
          fkl.d1 = k1.y; fkl.d2 = k1.z; fkl.F = (int)k1.w; fkl.negP = kc[9];
        }
        const int l0 = (Y.w & 63) - 1, l1 = ((Y.w >> 6) & 63) - 1;
        bool sok = false;
        int4 Pl = make_int4(0, 0, 0, 0);
        if (lane < ucount) {
          Pl = PSMEM ? lds_v4(P_sh + 16u * (unsigned)(ustart + lane)) : __ldcg(&P[ustart + lane]);
          sok = exact_mode || ((yt.hi[0] - Pl.x >= 0) & (yt.lo[0] - Pl.x < (int)p.W0) &
                               (yt.hi[1] - Pl.y >= 0) & (yt.lo[1] - Pl.y < (int)p.W1) &
                               (yt.hi[2] - Pl.z >= 0) & (yt.lo[2] - Pl.z < (int)p.W2));
        }
        // guard-band risk (dses_capi.cu): the source's fraction bucket on each
        // axis against the group's bitmaps; safe sources skip the near test
        bool safe = false;
        if (RISK && sok && !yt.pad[0]) {
          const unsigned* bm = p.risk + (size_t)(unit >> 16) * kRiskWords;
          const int sh = p.risk_shift;
          const unsigned w0 = __ldg(bm + (((unsigned)Pl.x >> (sh + 5)) & 31u));
          const unsigned w1 = __ldg(bm + 32 + (((unsigned)Pl.y >> (sh + 5)) & 31u));
          const unsigned w2 = __ldg(bm + 64 + (((unsigned)Pl.z >> (sh + 5)) & 31u));
          safe = (((w0 >> (((unsigned)Pl.x >> sh) & 31u)) | (w1 >> (((unsigned)Pl.y >> sh) & 31u)) |
                   (w2 >> (((unsigned)Pl.z >> sh) & 31u))) & 1u) == 0u;
        }
        const unsigned msafe = RISK ? __ballot_sync(0xffffffffu, safe) : 0u;
        const unsigned sm = __ballot_sync(0xffffffffu, sok);
        const unsigned mrisk = sm & ~msafe;
        const int nsafe = RISK ? __popc(msafe) : 0;
        // evaluated-pair statistic: a 32-bit per-warp counter (a 64-bit shared
        // add would be a CAS loop), folded into 64 bits once per rotation
        if (lane == 0)
          reds_add((uint32_t)__cvta_generic_to_shared(s_pairs) + 4u * (unsigned)warp,
                   (unsigned)__popc(sm) * (unsigned)yt.count);
        const int nsrc = __popc(sm);
        (void)nsafe;
        // opaque copy: keeps the stage base in a register (otherwise it is
        // re-derived from kernel parameters in every slot)
        uint32_t sbase;
        asm volatile("mov.u32 %0, %1;" : "=r"(sbase) : "r"(stage_sh));
        __syncwarp();  // the previous unit's slots have read the stage
        // safe sources first, then the rest
        if (sok) sts_v4(sbase + 16u * (unsigned)(!RISK ? __popc(sm & lanemask_lt)
                                                 : safe ? __popc(msafe & lanemask_lt)
                                                        : nsafe + __popc(mrisk & lanemask_lt)),
                        make_int4(Pl.x, Pl.y, Pl.z, ustart + lane));
        __syncwarp();
  #define DSES_SLOTS(GP)                                                                         \
  int t = 0;                                                                                   \
  if (RISK)                                                                                    \
    for (; t + 3 < nsafe; t += 4)                                                              \
      vote_slot<HSMEM, PSMEM, GP, 4, true>(p, fkl, R, P, hist, hist_sh, L, Y, l0, l1,            \
                                         sbase + 16u * (unsigned)t, j, lane, lanemask_lt);      \
  for (; t + 3 < nsrc; t += 4)                                                                 \
    vote_slot<HSMEM, PSMEM, GP, 4, false>(p, fkl, R, P, hist, hist_sh, L, Y, l0, l1,           \
                                          sbase + 16u * (unsigned)t, j, lane, lanemask_lt);     \
  for (; t < nsrc; t += 2) {                                                                   \
    if (t + 1 < nsrc)                                                                          \
      vote_slot<HSMEM, PSMEM, GP, 2, false>(p, fkl, R, P, hist, hist_sh, L, Y, l0, l1,         \
                                            sbase + 16u * (unsigned)t, j, lane, lanemask_lt);   \
    else                                                                                       \
      vote_slot<HSMEM, PSMEM, GP, 1, false>(p, fkl, R, P, hist, hist_sh, L, Y, l0, l1,         \
                                            sbase + 16u * (unsigned)t, j, lane, lanemask_lt);   \
  }
        if (gp == 0) { DSES_SLOTS(0) }
        else if (gp == 1) { DSES_SLOTS(1) }
        else { DSES_SLOTS(2) }
  #undef DSES_SLOTS
      }
      __syncthreads();  // units[] is rebuilt by the next round
      if (OVF) {
        gnext = ((int)ovf == b0) ? 1 : gmax;
        b0 = (int)ovf;
      } else {
        b0 += gmax;
      }
    }
    if (L.nrare > 0) {
      L.rechecks += flush_rare<HSMEM, PSMEM>(p, R, P, hist, hist_sh, L.rare_sh, L.nrare, lane) & 0xffffu;
      L.nrare = 0;
    }
    if (lane == 0) { st_pairs += s_pairs[warp]; s_pairs[warp] = 0; }
    __syncthreads();

    // ---- mode, pass 1: block maximum M of the histogram (packed 16-bit max
    //      per word) and the vote total
    unsigned mx = 0;
    for (int w = tid; w < nw4; w += nthreads) {
      // global slabs are only touched by atomics (L2) and these L1-bypassing accesses
      const uint4 v = HSMEM ? hist4[w] : __ldcg(&hist4[w]);
      if (p.count16) {
        // sum of the two 16-bit halves of a word: ((v * 0x10001) mod 2^32) >> 16
        st_votes += ((v.x * 0x10001u) >> 16) + ((v.y * 0x10001u) >> 16) +
                    ((v.z * 0x10001u) >> 16) + ((v.w * 0x10001u) >> 16);
        mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(v.x, v.y), __vmaxu2(v.z, v.w)));
      } else {
        st_votes += (unsigned long long)v.x + v.y + v.z + v.w;
        mx = max(mx, max(max(v.x, v.y), max(v.z, v.w)));
      }
    }
    if (p.count16) mx = max(mx & 0xffffu, mx >> 16);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = (int)mx;
    __syncthreads();
    int M = 0;
    for (int w = 0; w < nwarps; ++w) M = max(M, red[w]);
    // (no barrier: pass 2 writes red[32..95], red[0..31] is rewritten only
    // after the next rotation's barriers)
    // ---- pass 2: re-zero, and locate the smallest flat bin at M and the
    //      number of bins at M (_kernels.py:159-170); words without M are skipped
    int best = M, blin = INT_MAX, bties = 0;
    const unsigned MM = (unsigned)M * 0x10001u;
    for (int w = tid; w < nw4; w += nthreads) {
      const uint4 v = HSMEM ? hist4[w] : __ldcg(&hist4[w]);
      if ((v.x | v.y | v.z | v.w) == 0u) continue;
      if (HSMEM) hist4[w] = make_uint4(0, 0, 0, 0); else __stcg(&hist4[w], make_uint4(0, 0, 0, 0));
      if (M == 0) continue;
      const unsigned vv[4] = {v.x, v.y, v.z, v.w};
      if (p.count16) {
        // a half equals M iff the packed max of (v, MM) has a half == M and
        // v has that half; test cheaply via min(v ^ MM) over halves == 0
        const unsigned z = __vminu2(__vminu2(v.x ^ MM, v.y ^ MM), __vminu2(v.z ^ MM, v.w ^ MM));
        if ((z & 0xffffu) != 0u && (z >> 16) != 0u) continue;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int c = (int)((vv[h >> 1] >> ((h & 1) * 16)) & 0xffffu);
          if (c == M) { blin = min(blin, 8 * w + h); ++bties; }
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h)
          if ((int)vv[h] == M) { blin = min(blin, 4 * w + h); ++bties; }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      blin = min(blin, __shfl_xor_sync(0xffffffffu, blin, o));
      bties += __shfl_xor_sync(0xffffffffu, bties, o);
    }
    if (lane == 0) { red[32 + warp] = blin; red[64 + warp] = bties; }
    __syncthreads();
    if (warp == 0) {
      blin = lane < nwarps ? red[32 + lane] : INT_MAX;
      bties = lane < nwarps ? red[64 + lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        blin = min(blin, __shfl_xor_sync(0xffffffffu, blin, o));
        bties += __shfl_xor_sync(0xffffffffu, bties, o);
      }
      if (lane == 0) {
        const int64_t ro = REDO ? r - p.r_begin : rr;
        p.counts[ro] = best;
        p.lins[ro] = best > 0 ? blin : -1;
        p.ties[ro] = best > 0 ? bties : 0;
        s_rr = (long long)gridDim.x + (long long)atomicAdd(&p.stats[3], 1ull);
      }
    }
    __syncthreads();
    rr = s_rr;
  }

  // kernel statistics
  unsigned long long st_rechecks = L.rechecks;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st_pairs += __shfl_xor_sync(0xffffffffu, st_pairs, o);
    st_votes += __shfl_xor_sync(0xffffffffu, st_votes, o);
    st_rechecks += __shfl_xor_sync(0xffffffffu, st_rechecks, o);
  }
  if (lane == 0) {
    atomicAdd(&p.stats[0], st_pairs);
    atomicAdd(&p.stats[1], st_votes);
    atomicAdd(&p.stats[2], st_rechecks);
  }
}

// ===========================================================================
// Rotation-block kernel.  A block is a box of up to
// kMaxBlockRot neighbouring grid rotations (blk_s[0] x blk_s[1] x blk_s[2]
// along the Euler-index axes) inside the search's rotation range.  Every
// rotation R_t of the block moves a source point x by at most
//     |(R_t - Rc) x|_k <= sum_l |R_t,kl - Rc,kl| * max_unit |x_l|
// from its position under the block's centre rotation Rc (per source unit,
// in fixed-point units, + 3 for the two roundings), so the pairs that can
// vote for ANY rotation of the block are among the pairs inside the window
// widened by that bound at Rc.  The kernel
//   1. builds that candidate-pair list ONCE per block: the per-rotation
//      kernel's culling (unit boxes, group boxes, per-source tests) with the
//      widened windows, then one ballot per (source, group) and the candidate
//      lanes appended as entries i << jbits | j;
//   2. votes it for each rotation of the block: lane = one entry (no idle
//      lanes on out-of-window reference points), the same fixed-point bin
//      and guard band as the per-rotation kernel, and the per-source dedup
//      within the 32-entry segment: an entry compares its bin with the
//      entries of its earlier component mates (shuffles over the `off`
//      preceding lanes; mates of one source are contiguous in a run).
// Exact dedup needs every pair that can share (i, bin) -- dedup partners, i.e.
// points of one component -- in the same segment: a (source, group) run's
// entries never straddle a segment boundary (the rest of the segment is
// padded with the empty sentinel entry).  A segment holding a guard-band
// ("near") or split-component pair sends all its partnered pairs through the
// exact binary64 path (vote_exact: the reference's rule over the full near
// list).  A block whose list exceeds the CTA's slab, or whose widening
// exceeds 2^27 units, is left to vote_kernel (redo list).  Counts, bins and
// ties are those of the per-rotation kernel.

// The warp's open list segment is staged in shared memory (the warp's
// exact-path list area, unused while a block's list is built) and written to
// the CTA's slab, 32 entries at once, when full.  One (source, group) run
// never straddles two segments (so neither does a dedup component): a run
// that does not fit the open segment's room closes it (the rest padded with
// the empty sentinel entry).  A full slab sets the block's overflow flag.
__device__ __forceinline__ void flush_segment(const VoteParams& p, uint32_t buf_sh, int lane,
                                              uint32_t nseg_sh, uint32_t lovf_sh, unsigned slab,
                                              const int4& pad_entry, int& fill) {
  if (fill == 0) return;
  if (lane >= fill) sts_v4(buf_sh + 16u * (unsigned)lane, pad_entry);
  __syncwarp();
  const int4 e = lds_v4(buf_sh + 16u * (unsigned)lane);
  unsigned s = 0;
  if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(s) : "r"(nseg_sh) : "memory");
  s = __shfl_sync(0xffffffffu, s, 0);
  __syncwarp();  // every lane's read of the staging area before the next emit's writes
  fill = 0;
  if (32u * (s + 1u) > (unsigned)p.list_cap) {
    if (lane == 0) asm volatile("st.shared.u32 [%0], 1;" ::"r"(lovf_sh) : "memory");
    return;
  }
  __stcg(reinterpret_cast<int4*>(p.list) + (slab + 32u * s + (unsigned)lane), e);
}

// m = the warp's ballot of `mine`
__device__ __forceinline__ void emit_entries(const VoteParams& p, unsigned m, bool mine, const int4& entry,
                                             int lane, unsigned lanemask_lt, uint32_t buf_sh,
                                             uint32_t nseg_sh, uint32_t lovf_sh, unsigned slab,
                                             const int4& pad_entry, int& fill, unsigned& wcount) {
  const int cnt = __popc(m);
  wcount += (unsigned)cnt;
  if (cnt > 32 - fill) flush_segment(p, buf_sh, lane, nseg_sh, lovf_sh, slab, pad_entry, fill);  // warp-uniform
  if (mine) sts_v4(buf_sh + 16u * (unsigned)(fill + __popc(m & lanemask_lt)), entry);
  fill += cnt;
}

#ifndef DSES_BLOCK_THREADS
#define DSES_BLOCK_THREADS kVoteThreads
#endif
__global__ void __launch_bounds__(DSES_BLOCK_THREADS, 1) vote_blocks_kernel(const VoteParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = (int)lane_sr();
  constexpr int nthreads = DSES_BLOCK_THREADS, nwarps = nthreads >> 5;  // (launch_vote_blocks' launch)
  const int warp = tid >> 5;

  // the per-rotation kernel's layout (hsmem, psmem)
  size_t off = 0;
  unsigned* hist = reinterpret_cast<unsigned*>(smem);
  off += (size_t)p.hist_words * 4;
  int4* P = reinterpret_cast<int4*>(smem + off);
  off += (size_t)p.n_pad * 16;
  const int nxc = (p.nxt + 31) >> 5;
  int4* XB = reinterpret_cast<int4*>(smem + off);  // unit boxes, widened by the unit's motion bound
  int4* CB = XB + 2 * p.nxt;
  int4* DQ = CB + 2 * nxc;                          // per unit: the widening per axis
  off += (size_t)(p.nxt + nxc) * 32 + (size_t)p.nxt * 16;
  double* Rb = reinterpret_cast<double*>(smem + off);  // [kMaxBlockRot + 1][9]: block, centre
  off += kRotAreaBytes;
  int* red = reinterpret_cast<int*>(smem + off);
  off += 4 * 32 * 4;
  unsigned* units = reinterpret_cast<unsigned*>(smem + off);
  off += (size_t)p.unit_cap * 4;
  int2* rare = reinterpret_cast<int2*>(smem + off) + warp * kRare;
  off += (size_t)nwarps * kRare * 8;
  int4* stage = reinterpret_cast<int4*>(smem + off) + warp * 32;
  const uint32_t stage_sh = (uint32_t)__cvta_generic_to_shared(stage);

  int* s_nunits = red + 96;
  int* s_next = red + 97;
  int* s_ovf = red + 98;
  const unsigned lanemask_lt = lanemask_lt_sr();
  __shared__ __align__(16) unsigned kc[16];
  __shared__ int s_wide;                         // some unit's widening overflowed
  __shared__ int s_nseg;
  __shared__ int s_lovf;
  __shared__ long long s_rl[kMaxBlockRot];       // the current block's rotations ...
  __shared__ int s_nb;                           // ... their count (-1: done) ...
  __shared__ long long s_rc;                     // ... its centre rotation ...
  __shared__ int s_tc;                           // ... and the centre's place in s_rl (-1: none)
  __shared__ long long s_qa[6];                  // block queue: first a-part, a-parts, parts per axis, blocks
  __shared__ unsigned long long s_wst[32][2];    // per-warp (pairs, votes) statistics
  if (tid < 64) s_wst[tid >> 1][tid & 1] = 0;
  if (tid == 0) {
    kc[0] = p.W0; kc[1] = p.W1; kc[2] = p.W2; kc[3] = p.fmask; kc[4] = p.gthr;
    kc[5] = (unsigned)p.d1; kc[6] = (unsigned)p.d2; kc[7] = (unsigned)p.F;
    kc[8] = (uint32_t)__cvta_generic_to_shared(hist);
    kc[9] = 0u - (1u << p.F);
    kc[10] = (uint32_t)__cvta_generic_to_shared(P);
    kc[11] = (1u << p.jbits) - 1u;
    kc[12] = (unsigned)blockIdx.x * (unsigned)p.list_cap;  // this CTA's list slab (entry offset)
    kc[13] = g_dummy_sh;                                    // the dummy vote words
    kc[14] = kc[15] = 0u;
    g_exR = Rb;
    g_exP = P;
    g_exH = hist;
  }
  __syncthreads();
  // constants through shared memory: re-loaded where needed rather than
  // re-derived from the kernel parameters (register pressure at 64)
  const uint32_t hist_sh = kc[8];
  const uint32_t P_sh = kc[10];
  Lane L;
  asm volatile("mov.u32 %0, %1;" : "=r"(L.rare_sh) : "r"((uint32_t)__cvta_generic_to_shared(rare)));
  L.nrare = 0;
  L.rechecks = 0;

  uint4* hist4 = reinterpret_cast<uint4*>(hist);
  const int nw4 = p.hist_words >> 2;
  for (int w = tid; w < nw4; w += nthreads) hist4[w] = make_uint4(0, 0, 0, 0);

  const unsigned slab = kc[12];  // this CTA's list (entry offset)
  const uint32_t nseg_sh = (uint32_t)__cvta_generic_to_shared(&s_nseg);
  const uint32_t lovf_sh = (uint32_t)__cvta_generic_to_shared(&s_lovf);
  const unsigned jmask = kc[11];
  // list entries carry the reference point: (Yq.x, Yq.y, Yq.z, i << (jbits + 4) | j << 4 | c),
  // c = the number of earlier entries of the run in the point's dedup component
  // (15: split component / offset >= 15, exact path)
  const int ishift = p.ishift;
  const int4 pad_entry = make_int4(kNoRef, 0, 0, (int)((unsigned)p.m_pad << 4));  // never a candidate
  const int gmax = max(1, min(min(p.nyt, p.unit_cap / 4), p.unit_cap - p.nxt - 1));
  const bool masks = nxc > 1 && nxc <= 32;

  // blocks: boxes of blk_s[0] x blk_s[1] x blk_s[2] neighbouring grid
  // rotations (balanced parts of the Euler-index axes), restricted to
  // [r_begin, r_end), from a global queue (the first one static); thread 0
  // keeps the claim state, the rest read the block from shared memory (no
  // 64-bit loop state in every thread)
  long long bclaim = blockIdx.x;
  if (tid == 0) {  // the block queue's geometry: parts per axis, the a-parts that meet the range
    const int64_t n = 2 * p.rot.k + 1, n2 = n * n, pa = (n + p.blk_s[0] - 1) / p.blk_s[0];
    const int64_t a_lo = p.r_begin / n2, a_hi = (p.r_begin + p.r_count - 1) / n2;
    int64_t q0 = pa, q1 = -1;
    for (int64_t q = 0; q < pa; ++q)
      if ((q + 1) * n / pa > a_lo && q * n / pa <= a_hi) { q0 = min(q0, q); q1 = q; }
    s_qa[0] = q0;
    s_qa[1] = q1 - q0 + 1;
    s_qa[2] = pa;
    s_qa[3] = (n + p.blk_s[1] - 1) / p.blk_s[1];
    s_qa[4] = (n + p.blk_s[2] - 1) / p.blk_s[2];
    s_qa[5] = s_qa[1] * s_qa[3] * s_qa[4];  // blocks
  }
  for (;;) {
    if (tid == 0) {
      // the next non-empty block: the box's rotations inside [r_begin, r_end),
      // its centre and the centre's place among them (-1: outside the range);
      // per-axis indices in 32 bits (sides < 2^16), flat rotations in 64
      const int n = 2 * (int)p.rot.k + 1, pa = s_qa[2], pb = s_qa[3], pc = s_qa[4];
      const long long r_end = p.r_begin + p.r_count;
      int nb = -1;
      while (bclaim < s_qa[5]) {
        const int qa = (int)s_qa[0] + (int)(bclaim / (pb * pc)), qb = (int)((bclaim / pc) % pb),
                  qc = (int)(bclaim % pc);
        bclaim = (long long)gridDim.x + (long long)atomicAdd(&p.stats[3], 1ull);
        const int a0 = qa * n / pa, a1 = (qa + 1) * n / pa, b0 = qb * n / pb, b1 = (qb + 1) * n / pb,
                  c0 = qc * n / pc, c1 = (qc + 1) * n / pc;
        const long long rcen = ((long long)((a0 + a1 - 1) / 2) * n + (b0 + b1 - 1) / 2) * n + (c0 + c1 - 1) / 2;
        int cnt = 0, tc = -1;
        for (int a = a0; a < a1; ++a)
          for (int b = b0; b < b1; ++b) {
            const long long r0 = ((long long)a * n + b) * n;
            for (int c = c0; c < c1; ++c)
              if (r0 + c >= p.r_begin && r0 + c < r_end) {
                if (r0 + c == rcen) tc = cnt;
                s_rl[cnt++] = r0 + c;
              }
          }
        if (cnt > 0) {
          nb = cnt;
          s_rc = rcen;
          s_tc = tc;
          break;
        }
      }
      s_nb = nb;
      s_nseg = 0;
      s_lovf = 0;
      s_wide = 0;
    }
    __syncthreads();
    const int nb = s_nb;
    if (nb < 0) break;
    {
      const int tc = s_tc;  // the centre's place in the block (-1: outside the range)
      double* R = Rb + 9 * kMaxBlockRot;  // the centre rotation
      if (tid < 9) R[tid] = rotation_entry(p.rot, s_rc, tid);
      if (tid >= 32 && tid < 32 + 9 * nb) Rb[tid - 32] = rotation_entry(p.rot, s_rl[(tid - 32) / 9], (tid - 32) % 9);
      __syncthreads();
      // ---- A at the centre rotation: fixed-point points, and per unit the
      //      bound on its points' motion over the block's rotations,
      //      |(R_t - Rc) x|_k <= sum_l |R_t,kl - Rc,kl| max_unit |x_l|
      //      (fixed-point units, + 3 for the two roundings), and its box
      //      widened by that bound
      for (int a = warp; a < p.nxt; a += nwarps) {
        const int2 U = __ldg(reinterpret_cast<const int2*>(p.xt + a));
        const bool valid = lane < U.y;
        const int i = U.x + (valid ? lane : 0);
        int4 v = make_int4(0, 0, 0, 0);
        int ax0 = 0, ax1 = 0, ax2 = 0;
        if (valid) {
          const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
          v.x = __double2int_rn(dmul(rot_row(R, 0, x0, x1, x2), p.inv_s));
          v.y = __double2int_rn(dmul(rot_row(R, 1, x0, x1, x2), p.inv_s));
          v.z = __double2int_rn(dmul(rot_row(R, 2, x0, x1, x2), p.inv_s));
          sts_v4(P_sh + 16u * (unsigned)i, v);
          ax0 = (int)ceil(fabs(x0) * p.inv_s);
          ax1 = (int)ceil(fabs(x1) * p.inv_s);
          ax2 = (int)ceil(fabs(x2) * p.inv_s);
        }
        ax0 = __reduce_max_sync(0xffffffffu, ax0);
        ax1 = __reduce_max_sync(0xffffffffu, ax1);
        ax2 = __reduce_max_sync(0xffffffffu, ax2);
        int dq = 0;
        if (lane < 3) {  // axis `lane`
          double d = 0.0;
          for (int t = 0; t < nb; ++t) {
            const double* Rt = Rb + 9 * t + 3 * lane;
            const double* Rc = R + 3 * lane;
            d = fmax(d, fabs(Rt[0] - Rc[0]) * ax0 + fabs(Rt[1] - Rc[1]) * ax1 + fabs(Rt[2] - Rc[2]) * ax2);
          }
          // (a widening beyond 2^27 units -- huge steps -- leaves the block to vote_kernel)
          dq = d < 134217728.0 ? (int)ceil(d * (1.0 + 1e-9)) + 3 : -1;
        }
        const int dq0 = __shfl_sync(0xffffffffu, dq, 0), dq1 = __shfl_sync(0xffffffffu, dq, 1),
                  dq2 = __shfl_sync(0xffffffffu, dq, 2);
        const int4 blo = make_int4(__reduce_min_sync(0xffffffffu, valid ? v.x : INT_MAX) - dq0,
                                   __reduce_min_sync(0xffffffffu, valid ? v.y : INT_MAX) - dq1,
                                   __reduce_min_sync(0xffffffffu, valid ? v.z : INT_MAX) - dq2, U.x);
        const int4 bhi = make_int4(__reduce_max_sync(0xffffffffu, valid ? v.x : INT_MIN) + dq0,
                                   __reduce_max_sync(0xffffffffu, valid ? v.y : INT_MIN) + dq1,
                                   __reduce_max_sync(0xffffffffu, valid ? v.z : INT_MIN) + dq2, U.x + U.y);
        if (lane == 0) {
          XB[2 * a] = blo;
          XB[2 * a + 1] = bhi;
          DQ[a] = make_int4(dq0, dq1, dq2, 0);
          if ((dq0 | dq1 | dq2) < 0) s_wide = 1;
        }
      }
      __syncthreads();
      for (int c = warp; c < nxc; c += nwarps) {
        const int t = 32 * c + lane;
        const bool valid = t < p.nxt;
        int4 blo = valid ? XB[2 * t] : make_int4(INT_MAX, INT_MAX, INT_MAX, 0);
        int4 bhi = valid ? XB[2 * t + 1] : make_int4(INT_MIN, INT_MIN, INT_MIN, 0);
        blo.x = __reduce_min_sync(0xffffffffu, blo.x);
        blo.y = __reduce_min_sync(0xffffffffu, blo.y);
        blo.z = __reduce_min_sync(0xffffffffu, blo.z);
        bhi.x = __reduce_max_sync(0xffffffffu, bhi.x);
        bhi.y = __reduce_max_sync(0xffffffffu, bhi.y);
        bhi.z = __reduce_max_sync(0xffffffffu, bhi.z);
        if (lane == 0) { CB[2 * c] = blo; CB[2 * c + 1] = bhi; }
      }
      __syncthreads();

      // ---- build the block's list (rounds of reference groups, as vote_kernel,
      //      against the widened unit boxes)
      int fill = 0;
      const bool wide = s_wide != 0;  // block-uniform
      if (wide && tid == 0) s_lovf = 1;  // (read after the build's barriers)
      unsigned wcount = 0;
      for (int b0 = 0, gnext = gmax; b0 < (wide ? 0 : p.nyt);) {
        const int b1 = min(p.nyt, b0 + gnext);
        if (tid == 0) { *s_nunits = 0; *s_next = 0; *s_ovf = b1; }
        const int cap_u = p.unit_cap - gmax;
        unsigned* gmask = units + cap_u;
        if (masks)
          for (int k = tid; k < b1 - b0; k += nthreads) {
            const YTile yg = load_ytile(p.yt, b0 + k);
            unsigned mk = 0;
            for (int c = 0; c < nxc; ++c)
              if (boxes_meet(p, yg, CB[2 * c], CB[2 * c + 1])) mk |= 1u << c;
            gmask[k] = mk;
          }
        __syncthreads();
        for (int b = b0 + warp; b < b1; b += nwarps) {
          const YTile yt = load_ytile(p.yt, b);
          for (int a0 = 0; a0 < p.nxt; a0 += 32) {
            if (masks ? !((gmask[b - b0] >> (a0 >> 5)) & 1u)
                      : (nxc > 1 && !boxes_meet(p, yt, CB[2 * (a0 >> 5)], CB[2 * (a0 >> 5) + 1])))
              continue;
            const int a = a0 + lane;
            const bool ov = a < p.nxt && boxes_meet(p, yt, XB[2 * a], XB[2 * a + 1]);
            const unsigned m = __ballot_sync(0xffffffffu, ov);
            if (m) {
              int slot = 0;
              if (lane == 0) {
                slot = atomicAdd(s_nunits, __popc(m));
                if (slot + __popc(m) > cap_u) atomicMin(s_ovf, b);
              }
              slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(m & lanemask_lt);
              if (ov && slot < cap_u) units[slot] = ((unsigned)b << 16) | (unsigned)a;
            }
          }
        }
        __syncthreads();
        const int nunits = min(*s_nunits, cap_u);
        const unsigned ovf = (unsigned)*s_ovf;
        for (int u = 0;; ++u) {
          if (lane == 0) u = atomicAdd(s_next, 1);
          u = __shfl_sync(0xffffffffu, u, 0);
          if (u >= nunits) break;
          const unsigned unit = units[u];
          if ((unit >> 16) >= ovf) continue;  // warp-uniform
          const YTile yt = load_ytile(p.yt, (int)(unit >> 16));
          const int2 U = __ldg(reinterpret_cast<const int2*>(p.xt + (unit & 0xffffu)));
          const bool valid = lane < yt.count;
          const int j = yt.start + (valid ? lane : 0);
          int4 Y = __ldg(&p.yq[j]);
          if (!valid) Y = make_int4(kNoRef, 0, 0, 0);
          const int4 dq = DQ[unit & 0xffffu];  // the unit's widening
          // the entry's low 4 bits: the number of earlier entries of the same
          // run (source) in the point's dedup component -- the lanes it must
          // compare bins with -- or 15 (split component / offset >= 15: exact)
          const unsigned offs = (Y.w & kSplitFlag) ? 15u : (unsigned)min((Y.w >> kCompOffShift) & 15, 15);
          const unsigned jw = ((unsigned)j << 4) | (offs == 15u ? 15u : 0u);
          const unsigned cmask = offs == 15u ? 0u : lanemask_lt & (0xffffffffu << max(lane - (int)offs, 0));
          const int y0 = (int)((unsigned)Y.x + (unsigned)dq.x), y1 = (int)((unsigned)Y.y + (unsigned)dq.y),
                    y2 = (int)((unsigned)Y.z + (unsigned)dq.z);
          const unsigned Wp0 = p.W0 + 2u * (unsigned)dq.x, Wp1 = p.W1 + 2u * (unsigned)dq.y,
                         Wp2 = p.W2 + 2u * (unsigned)dq.z;
          bool sok = false;
          int4 Pl = make_int4(0, 0, 0, 0);
          if (lane < U.y) {
            Pl = lds_v4(P_sh + 16u * (unsigned)(U.x + lane));
            sok = (yt.hi[0] - Pl.x >= -dq.x) & (yt.lo[0] - Pl.x < (int)p.W0 + dq.x) &
                  (yt.hi[1] - Pl.y >= -dq.y) & (yt.lo[1] - Pl.y < (int)p.W1 + dq.y) &
                  (yt.hi[2] - Pl.z >= -dq.z) & (yt.lo[2] - Pl.z < (int)p.W2 + dq.z);
          }
          const unsigned sm = __ballot_sync(0xffffffffu, sok);
          const int nsrc = __popc(sm);
          __syncwarp();
          if (sok) sts_v4(stage_sh + 16u * (unsigned)__popc(sm & lanemask_lt),
                          make_int4(Pl.x, Pl.y, Pl.z, U.x + lane));
          __syncwarp();
          // two staged sources per step (a slab overflow only stops the
          // writes: the block goes to vote_kernel)
          for (int t = 0; t < nsrc; t += 2) {
            const int4 P0 = lds_v4(stage_sh + 16u * (unsigned)t);
            const int4 P1 = lds_v4(stage_sh + 16u * (unsigned)min(t + 1, 31));
            const bool c0 = ((unsigned)y0 - (unsigned)P0.x < Wp0) & ((unsigned)y1 - (unsigned)P0.y < Wp1) &
                            ((unsigned)y2 - (unsigned)P0.z < Wp2);
            const bool c1 = ((unsigned)y0 - (unsigned)P1.x < Wp0) & ((unsigned)y1 - (unsigned)P1.y < Wp1) &
                            ((unsigned)y2 - (unsigned)P1.z < Wp2) & (t + 1 < nsrc);
            const unsigned m0 = __ballot_sync(0xffffffffu, c0), m1 = __ballot_sync(0xffffffffu, c1);
            if (m0)
              emit_entries(p, m0, c0, make_int4(Y.x, Y.y, Y.z, (int)(((unsigned)P0.w << ishift) | jw |
                                                                     (unsigned)__popc(m0 & cmask))), lane,
                           lanemask_lt, L.rare_sh, nseg_sh, lovf_sh, slab, pad_entry, fill, wcount);
            if (m1)
              emit_entries(p, m1, c1, make_int4(Y.x, Y.y, Y.z, (int)(((unsigned)P1.w << ishift) | jw |
                                                                     (unsigned)__popc(m1 & cmask))), lane,
                           lanemask_lt, L.rare_sh, nseg_sh, lovf_sh, slab, pad_entry, fill, wcount);
          }
        }
        __syncthreads();
        gnext = ((int)ovf == b0) ? 1 : gmax;
        b0 = (int)ovf;
      }
      flush_segment(p, L.rare_sh, lane, nseg_sh, lovf_sh, slab, pad_entry, fill);
      __syncthreads();
      if (s_lovf) {  // left to vote_kernel
        if (tid < nb) p.redo[atomicAdd(p.redo_n, 1ull)] = s_rl[tid];
      } else {
        const int nseg = s_nseg;
        if (lane == 0) s_wst[warp][0] += (unsigned long long)wcount * (unsigned long long)nb;
        for (int t0 = 0; t0 < nb; ++t0) {
          // the centre first when it is in the block: P holds it
          const int t = tc < 0 ? t0 : (t0 == 0 ? tc : (t0 <= tc ? t0 - 1 : t0));
          const double* Rt = Rb + 9 * t;
          if (t != tc) {
            for (int i = tid; i < p.n; i += nthreads) {
              const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
              sts_v4(P_sh + 16u * (unsigned)i,
                     make_int4(__double2int_rn(dmul(rot_row(Rt, 0, x0, x1, x2), p.inv_s)),
                               __double2int_rn(dmul(rot_row(Rt, 1, x0, x1, x2), p.inv_s)),
                               __double2int_rn(dmul(rot_row(Rt, 2, x0, x1, x2), p.inv_s)), 0));
            }
          }
          if (tid == 0) g_exR = Rt;
          __syncthreads();
          // ---- vote the list: lane = one entry
          FastK fk;
          {
            const uint4 k0 = *reinterpret_cast<const uint4*>(kc);
            const uint4 k1 = *reinterpret_cast<const uint4*>(kc + 4);
            fk.W0 = k0.x; fk.W1 = k0.y; fk.W2 = k0.z; fk.fmask = k0.w;
            fk.gthr = k1.x; fk.d1 = k1.y; fk.d2 = k1.z; fk.F = (int)k1.w; fk.negP = kc[9];
          }
          const uint32_t dummy_sh = kc[13] + 4u * (unsigned)lane;  // this lane's sink word
          // (the next segment's entry is loaded one iteration ahead: the list
          // comes from L2; one segment per warp past the list's end is read and
          // unused -- the allocation has kBlockListSlack entries after the last slab)
          const int4* qn = reinterpret_cast<const int4*>(p.list) + (slab + 32u * (unsigned)warp + (unsigned)lane);
          int4 en_next = __ldcg(qn);
          for (int sg = warp; sg < nseg; sg += nwarps) {
            const int4 Y = en_next;  // the entry: the reference point and (i, j, o)
            qn += 32 * nwarps;
            en_next = __ldcg(qn);
            const unsigned ew = (unsigned)Y.w, e = ew >> 4;
            const int i = (int)(ew >> ishift);
            const int4 Pi = lds_v4(P_sh + 16u * (unsigned)i);
            const unsigned u0 = (unsigned)(Y.x - Pi.x), u1 = (unsigned)(Y.y - Pi.y), u2 = (unsigned)(Y.z - Pi.z);
            const bool cand = (u0 < fk.W0) & (u1 < fk.W1) & (u2 < fk.W2);
            const unsigned q0 = u0 >> fk.F, q1 = u1 >> fk.F, q2 = u2 >> fk.F;
            const unsigned gthr = (ew & 15u) == 15u ? 0xffffffffu : fk.gthr;
            const bool near = cand & (__vimin3_u32(u0 + q0 * fk.negP, u1 + q1 * fk.negP, u2 + q2 * fk.negP) < gthr);
            const unsigned lin = (q0 * fk.d1 + q1) * fk.d2 + q2;
            if (!__any_sync(0xffffffffu, near)) {
              // every candidate decided: a (source, bin) votes once, by its lowest
              // lane.  Lanes that can share it are entries of one component for
              // one source, contiguous in the segment: the entry's `c` (its low
              // 4 bits, set by the build) earlier lanes are exactly its mates
              const int c = (int)(ew & 15u);
              const int key = cand ? (int)lin : -1;
              const int dmax = __reduce_max_sync(0xffffffffu, cand ? c : 0);
              bool ok = cand;
              if (dmax > 0) {  // (warp-uniform) most segments need one step, a few more
                ok &= !(__shfl_up_sync(0xffffffffu, key, 1) == key && c >= 1);
#pragma unroll 1
                for (int d = 2; d <= dmax; ++d) ok &= !(__shfl_up_sync(0xffffffffu, key, d) == key && c >= d);
              }
              const uint32_t a = ok ? hist_sh + ((lin + lin) & ~3u) : dummy_sh;
              reds_add(a, __funnelshift_l(0u, 1u, lin << 4));
            } else {
              // a near / split pair in the segment: its partners' bins are not
              // known exactly -- every partnered candidate takes the exact path
              const int j = (int)(e & jmask);
              const bool def = near | (cand && (__ldg(&p.yq[j].w) & kPartFlag) != 0);
              vote_if<true>(hist, hist_sh, lin, cand & !def, (unsigned)p.nbins);
              const unsigned dm = __ballot_sync(0xffffffffu, def);
              if (dm) defer_pairs<true, true>(p, hist_sh, L, dm, def, i, j, lane, lanemask_lt);
            }
          }
          if (L.nrare > 0) {
            L.rechecks += flush_rare<true, true>(p, Rt, P, hist, hist_sh, L.rare_sh, L.nrare, lane) & 0xffffu;
            L.nrare = 0;
          }
          __syncthreads();
          // ---- mode (vote_kernel's two passes)
          unsigned mx = 0, nv = 0;
          for (int w = tid; w < nw4; w += nthreads) {
            const uint4 v = hist4[w];
            nv += ((v.x * 0x10001u) >> 16) + ((v.y * 0x10001u) >> 16) + ((v.z * 0x10001u) >> 16) +
                  ((v.w * 0x10001u) >> 16);
            mx = __vmaxu2(mx, __vmaxu2(__vmaxu2(v.x, v.y), __vmaxu2(v.z, v.w)));
          }
          mx = max(mx & 0xffffu, mx >> 16);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            nv += __shfl_xor_sync(0xffffffffu, nv, o);
          }
          if (lane == 0) { red[warp] = (int)mx; s_wst[warp][1] += nv; }
          __syncthreads();
          // (no barrier after reading the maxima: pass 2 writes red[32..95], and
          // red[0..31] is rewritten only after the next rotation's vote barrier)
          const int M = (int)__reduce_max_sync(0xffffffffu, lane < nwarps ? (unsigned)red[lane] : 0u);
          int blin = INT_MAX, bties = 0;
          const unsigned MM = (unsigned)M * 0x10001u;
          for (int w = tid; w < nw4; w += nthreads) {
            const uint4 v = hist4[w];
            if ((v.x | v.y | v.z | v.w) == 0u) continue;
            hist4[w] = make_uint4(0, 0, 0, 0);
            if (M == 0) continue;
            const unsigned z = __vminu2(__vminu2(v.x ^ MM, v.y ^ MM), __vminu2(v.z ^ MM, v.w ^ MM));
            if ((z & 0xffffu) != 0u && (z >> 16) != 0u) continue;
            const unsigned vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
              const int c = (int)((vv[h >> 1] >> ((h & 1) * 16)) & 0xffffu);
              if (c == M) { blin = min(blin, 8 * w + h); ++bties; }
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            blin = min(blin, __shfl_xor_sync(0xffffffffu, blin, o));
            bties += __shfl_xor_sync(0xffffffffu, bties, o);
          }
          if (lane == 0) { red[32 + warp] = blin; red[64 + warp] = bties; }
          __syncthreads();
          if (warp == 0) {
            blin = lane < nwarps ? red[32 + lane] : INT_MAX;
            bties = lane < nwarps ? red[64 + lane] : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              blin = min(blin, __shfl_xor_sync(0xffffffffu, blin, o));
              bties += __shfl_xor_sync(0xffffffffu, bties, o);
            }
            if (lane == 0) {
              const int64_t ro = s_rl[t] - p.r_begin;
              p.counts[ro] = M;
              p.lins[ro] = M > 0 ? blin : -1;
              p.ties[ro] = M > 0 ? bties : 0;
            }
          }
          __syncthreads();
        }
      }
    }
    __syncthreads();  // s_lo / s_nb are rewritten for the next block
  }

  unsigned st_rechecks = L.rechecks;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) st_rechecks += __shfl_xor_sync(0xffffffffu, st_rechecks, o);
  if (lane == 0) {
    atomicAdd(&p.stats[0], s_wst[warp][0]);
    atomicAdd(&p.stats[1], s_wst[warp][1]);
    atomicAdd(&p.stats[2], (unsigned long long)st_rechecks);
  }
}

size_t vote_smem_bytes(const VoteParams& p, bool hsmem, bool psmem, int threads) {
  size_t b = 0;
  if (hsmem) b += (size_t)p.hist_words * 4;
  if (psmem) b += (size_t)p.n_pad * 16;
  b += (size_t)(p.nxt + (p.nxt + 31) / 32) * 32 + (size_t)p.nxt * 16 + kRotAreaBytes + 4 * 32 * 4 +
       (size_t)p.unit_cap * 4;  // (unit boxes, chunk boxes, the block kernel's per-unit widening, ...)
  b += (size_t)(threads / 32) * kRare * 8;
  b += (size_t)(threads / 32) * 32 * 16;  // per-warp staged sources
  return b;
}

// The dynamic shared-memory limit of each instantiation is raised ONCE per
// device to the opt-in maximum (minus its static shared memory) and never
// lowered: plan construction on one thread and launches on another must not
// race on this process-wide attribute (a lowered limit between another
// thread's set and launch would fail that launch).
template <bool H, bool PS, bool RK, bool RD = false>
static cudaError_t raise_smem_limit() {
  static std::once_flag once[64];
  static cudaError_t err[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    int optin = 0;
    cudaFuncAttributes a{};
    err[dev] = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (err[dev] == cudaSuccess) err[dev] = cudaFuncGetAttributes(&a, vote_kernel<H, PS, RK, RD>);
    if (err[dev] == cudaSuccess)
      err[dev] = cudaFuncSetAttribute(vote_kernel<H, PS, RK, RD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - (int)a.sharedSizeBytes);
  });
  return err[dev];
}

cudaError_t launch_vote(const VoteParams& p, bool hsmem, bool psmem, int grid, int threads,
                        cudaStream_t stream) {
  const size_t smem = vote_smem_bytes(p, hsmem, psmem, threads);
  const bool risk = p.risk_shift != 0;
  cudaError_t e;
#define DSES_LAUNCH(H, PS, RK)                      \
  e = raise_smem_limit<H, PS, RK>();                \
  if (e != cudaSuccess) return e;                   \
  vote_kernel<H, PS, RK><<<grid, threads, smem, stream>>>(p);
  if (hsmem && psmem) { if (risk) { DSES_LAUNCH(true, true, true) } else { DSES_LAUNCH(true, true, false) } }
  else if (hsmem) { DSES_LAUNCH(true, false, false) }
  else if (psmem) { DSES_LAUNCH(false, true, false) }
  else { DSES_LAUNCH(false, false, false) }
#undef DSES_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_vote_redo(const VoteParams& p, int grid, int threads, cudaStream_t stream) {
  const cudaError_t e = raise_smem_limit<true, true, false, true>();
  if (e != cudaSuccess) return e;
  vote_kernel<true, true, false, true><<<grid, threads, vote_smem_bytes(p, true, true, threads), stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_vote_blocks(const VoteParams& p, int grid, int threads, cudaStream_t stream) {
  static std::once_flag once[64];
  static cudaError_t err[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    int optin = 0;
    cudaFuncAttributes a{};
    err[dev] = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (err[dev] == cudaSuccess) err[dev] = cudaFuncGetAttributes(&a, vote_blocks_kernel);
    if (err[dev] == cudaSuccess)
      err[dev] = cudaFuncSetAttribute(vote_blocks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - (int)a.sharedSizeBytes);
  });
  if (err[dev] != cudaSuccess) return err[dev];
  threads = DSES_BLOCK_THREADS;
  vote_blocks_kernel<<<grid, threads, vote_smem_bytes(p, true, true, threads), stream>>>(p);
  return cudaGetLastError();
}

// Static shared memory of the vote kernel (kc[], exact-path pointers, ...):
// the dynamic part is sized against opt-in limit minus this.
size_t vote_static_smem() {
  cudaFuncAttributes a{};
  size_t m = 0;
  if (cudaFuncGetAttributes(&a, vote_kernel<true, true, true>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_kernel<true, true, false>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_kernel<true, false, false>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_kernel<false, true, false>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_kernel<false, false, false>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_blocks_kernel) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  if (cudaFuncGetAttributes(&a, vote_kernel<true, true, false, true>) == cudaSuccess) m = std::max(m, a.sharedSizeBytes);
  return m;
}

int vote_max_ctas_per_sm(const VoteParams& p, bool hsmem, bool psmem, int threads) {
  const size_t smem = vote_smem_bytes(p, hsmem, psmem, threads);
  const bool risk = p.risk_shift != 0;
  int n = 0;
  cudaError_t e;
#define DSES_OCC(H, PS, RK)                                                                \
  e = raise_smem_limit<H, PS, RK>();                                                       \
  if (e == cudaSuccess)                                                                    \
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vote_kernel<H, PS, RK>, threads, smem);
  if (hsmem && psmem) { if (risk) { DSES_OCC(true, true, true) } else { DSES_OCC(true, true, false) } }
  else if (hsmem) { DSES_OCC(true, false, false) }
  else if (psmem) { DSES_OCC(false, true, false) }
  else { DSES_OCC(false, false, false) }
#undef DSES_OCC
  return e == cudaSuccess ? n : 0;
}

}  // namespace dses
