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

constexpr int kUnitCap = 4096;  // (reference tile, source unit) work units per round

// Rotated sphere (centre +- radius, a rotation preserves |x - c|) of a source
// tile as a fixed-point box; .w carries the tile's point range.
__device__ __forceinline__ void tile_box(const VoteParams& p, const double* R, const XTile& t,
                                         bool exact_mode, int4& lo, int4& hi) {
  if (exact_mode) {
    lo = make_int4(INT_MIN / 4, INT_MIN / 4, INT_MIN / 4, t.start);
    hi = make_int4(INT_MAX / 4, INT_MAX / 4, INT_MAX / 4, t.start + t.count);
    return;
  }
  const int c0 = __double2int_rn(rot_row(R, 0, t.c[0], t.c[1], t.c[2]) * p.inv_s);
  const int c1 = __double2int_rn(rot_row(R, 1, t.c[0], t.c[1], t.c[2]) * p.inv_s);
  const int c2 = __double2int_rn(rot_row(R, 2, t.c[0], t.c[1], t.c[2]) * p.inv_s);
  lo = make_int4(c0 - t.rad, c1 - t.rad, c2 - t.rad, t.start);
  hi = make_int4(c0 + t.rad, c1 + t.rad, c2 + t.rad, t.start + t.count);
}

// Can a source box [lo, hi] and the reference tile bbox produce u = Yq - Pq in [0, W)?
__device__ __forceinline__ bool boxes_meet(const VoteParams& p, const YTile& yt, const int4& lo,
                                           const int4& hi) {
  return (yt.hi[0] - lo.x >= 0) & (yt.lo[0] - hi.x < (int)p.W0) & (yt.hi[1] - lo.y >= 0) &
         (yt.lo[1] - hi.y < (int)p.W1) & (yt.hi[2] - lo.z >= 0) & (yt.lo[2] - hi.z < (int)p.W2);
}

// One source point i against the warp's 32 reference points (one per lane).
// Branch-free fast path; the rare guard-band re-bin and the rare
// out-of-tile dedup are divergent branches entered only when some lane needs
// them.  Dedup (_kernels.py:153-158): the vote (i, j) is dropped when a near
// neighbour j' < j lands in the same bin for the same i; in-tile neighbours
// are other lanes of this warp, so their bins arrive by shuffle.
template <bool PSMEM>
__device__ __forceinline__ void vote_slot(const VoteParams& p, const double* R, const int4* P,
                                          unsigned* hist, const int4& Y, int j, int lane, int i,
                                          unsigned& votes, unsigned& rechecks) {
  const int4 Pi = PSMEM ? P[i] : __ldcg(&P[i]);
  const int u0 = Y.x - Pi.x, u1 = Y.y - Pi.y, u2 = Y.z - Pi.z;
  const bool cand = ((unsigned)u0 < p.W0) & ((unsigned)u1 < p.W1) & ((unsigned)u2 < p.W2);
  if (!__any_sync(0xffffffffu, cand)) return;
  const unsigned g2 = 2u * kGuard;
  const bool near = cand & ((((unsigned)u0 & p.fmask) < g2) | (((unsigned)u1 & p.fmask) < g2) |
                            (((unsigned)u2 & p.fmask) < g2));
  bool in = cand & !near & ((unsigned)u0 < p.D0) & ((unsigned)u1 < p.D1) & ((unsigned)u2 < p.D2);
  int lin = ((u0 >> p.F) * p.d1 + (u1 >> p.F)) * p.d2 + (u2 >> p.F);
  if (__any_sync(0xffffffffu, near)) {
    if (near) {
      ++rechecks;
      const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
      in = exact_bin(p, rot_row(R, 0, x0, x1, x2), rot_row(R, 1, x0, x1, x2),
                     rot_row(R, 2, x0, x1, x2), p.ys + 3 * j, &lin);
    }
  }
  const int key = in ? lin : -1;
  const int l0 = (Y.w & 63) - 1, l1 = ((Y.w >> 6) & 63) - 1;
  const int k0 = __shfl_sync(0xffffffffu, key, l0 & 31);
  const int k1 = __shfl_sync(0xffffffffu, key, l1 & 31);
  bool dup = in & (((l0 >= 0) & (k0 == key)) | ((l1 >= 0) & (k1 == key)));
  const bool far = in & !dup & ((Y.w >> 12) & 1);
  if (__any_sync(0xffffffffu, far)) {
    if (far) {
      const int e1 = p.near_off[j + 1];
      for (int k = p.near_off[j]; k < e1 && !dup; ++k) {
        const int jj = p.near_idx[k];
        int lin2;
        dup = pair_bin(p, R, Pi, i, p.yq[jj], jj, &lin2, rechecks) && lin2 == lin;
      }
    }
  }
  if (in & !dup) {
    ++votes;
    if (p.count16) atomicAdd(&hist[lin >> 1], (lin & 1) ? 0x10000u : 1u);
    else atomicAdd(&hist[lin], 1u);
  }
}

template <bool HSMEM, bool PSMEM>
__global__ void __launch_bounds__(kVoteThreads, 1) vote_kernel(const VoteParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nthreads = blockDim.x, nwarps = nthreads >> 5, warp = tid >> 5;

  size_t off = 0;
  unsigned* hist;
  if (HSMEM) { hist = reinterpret_cast<unsigned*>(smem); off += (size_t)p.hist_words * 4; }
  else hist = p.hist_global + (size_t)blockIdx.x * p.hist_words;
  int4* P;
  if (PSMEM) { P = reinterpret_cast<int4*>(smem + off); off += (size_t)p.n * 16; }
  else P = p.p_global + (size_t)blockIdx.x * p.n_pad;
  int4* XB = reinterpret_cast<int4*>(smem + off);  // [2*nxt] rotated unit boxes (lo, hi)
  off += (size_t)p.nxt * 32;
  int4* XS = reinterpret_cast<int4*>(smem + off);  // [2*nxs] rotated sub-tile boxes
  off += (size_t)p.nxs * 32;
  double* R = reinterpret_cast<double*>(smem + off);
  off += 16 * 8;
  int* red = reinterpret_cast<int*>(smem + off);    // [3 * 32] reduction scratch + counters
  off += 4 * 32 * 4;
  int* units = reinterpret_cast<int*>(smem + off);  // [kUnitCap] overlapping tile pairs
  int* s_nunits = red + 96;
  int* s_next = red + 97;
  const unsigned lanemask_lt = (1u << lane) - 1u;

  uint4* hist4 = reinterpret_cast<uint4*>(hist);
  const int nw4 = p.hist_words >> 2;
  for (int w = tid; w < nw4; w += nthreads) {
    if (HSMEM) hist4[w] = make_uint4(0, 0, 0, 0); else __stcg(&hist4[w], make_uint4(0, 0, 0, 0));
  }

  unsigned long long st_pairs = 0;
  unsigned st_votes = 0, st_rechecks = 0;
  const bool exact_mode = (p.F == 0);
  const int npairs = p.nyt * p.nxt;

  for (int64_t rr = blockIdx.x; rr < p.r_count; rr += gridDim.x) {
    const int64_t r = p.r_begin + rr;
    if (tid < 9) R[tid] = rotation_entry(p.rot, r, tid);
    __syncthreads();

    // ---- A: rotated source points in fixed point (fp64, the reference's op
    //      order) and rotated unit / sub-tile boxes
    for (int i = tid; i < p.n; i += nthreads) {
      const double x0 = p.xs[3 * i], x1 = p.xs[3 * i + 1], x2 = p.xs[3 * i + 2];
      int4 q = make_int4(0, 0, 0, 0);
      if (!exact_mode) {
        q.x = __double2int_rn(dmul(rot_row(R, 0, x0, x1, x2), p.inv_s));
        q.y = __double2int_rn(dmul(rot_row(R, 1, x0, x1, x2), p.inv_s));
        q.z = __double2int_rn(dmul(rot_row(R, 2, x0, x1, x2), p.inv_s));
      }
      if (PSMEM) P[i] = q; else __stcg(&P[i], q);
    }
    for (int t = tid; t < p.nxt + p.nxs; t += nthreads) {
      int4 lo, hi;
      if (t < p.nxt) {
        tile_box(p, R, p.xt[t], exact_mode, lo, hi);
        XB[2 * t] = lo;
        XB[2 * t + 1] = hi;
      } else {
        tile_box(p, R, p.xsub[t - p.nxt], exact_mode, lo, hi);
        XS[2 * (t - p.nxt)] = lo;
        XS[2 * (t - p.nxt) + 1] = hi;
      }
    }
    __syncthreads();

    // ---- B: votes, in rounds of at most kUnitCap (reference tile, source unit) pairs.
    //  B1  threads test tile pairs; overlapping ones are compacted into `units`;
    //  B2  warps take units dynamically: lane = reference point j (registers);
    //      lanes 0..7 test the unit's sub-tiles, then each surviving sub-tile's
    //      points i are broadcast from shared memory, one vote_slot per i.
    for (int base = 0; base < npairs; base += kUnitCap) {
      if (tid == 0) { *s_nunits = 0; *s_next = 0; }
      __syncthreads();
      const int lim = min(kUnitCap, npairs - base);
      for (int k0 = 0; k0 < lim; k0 += nthreads) {
        const int k = k0 + tid;
        bool ov = false;
        int unit = 0;
        if (k < lim) {
          unit = base + k;
          const int b = unit / p.nxt, a = unit - b * p.nxt;
          ov = exact_mode || boxes_meet(p, p.yt[b], XB[2 * a], XB[2 * a + 1]);
        }
        const unsigned m = __ballot_sync(0xffffffffu, ov);
        if (m) {
          int slot = 0;
          if (lane == 0) slot = atomicAdd(s_nunits, __popc(m));
          slot = __shfl_sync(0xffffffffu, slot, 0);
          if (ov) units[slot + __popc(m & lanemask_lt)] = unit;
        }
      }
      __syncthreads();
      const int nunits = *s_nunits;
      for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(s_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= nunits) break;
        const int unit = units[u];
        const int b = unit / p.nxt, a = unit - b * p.nxt;
        const YTile yt = p.yt[b];
        const bool valid = lane < yt.count;
        const int j = yt.start + (valid ? lane : 0);
        int4 Y = p.yq[j];
        if (!valid) { Y.x = INT_MIN / 2; Y.w = 0; }  // never a candidate
        const XTile& U = p.xt[a];
        const int nsub = U.nsub, sub0 = U.sub;
        bool sok = false;
        if (lane < nsub) sok = exact_mode || boxes_meet(p, yt, XS[2 * (sub0 + lane)], XS[2 * (sub0 + lane) + 1]);
        unsigned sm = __ballot_sync(0xffffffffu, sok);
        while (sm) {
          const int s = sub0 + __ffs(sm) - 1;
          sm &= sm - 1;
          const int i0 = XS[2 * s].w, i1 = XS[2 * s + 1].w;
          if (lane == 0) st_pairs += (unsigned long long)(i1 - i0) * yt.count;
          for (int i = i0; i < i1; ++i)
            vote_slot<PSMEM>(p, R, P, hist, Y, j, lane, i, st_votes, st_rechecks);
        }
      }
      __syncthreads();  // units[] is rebuilt by the next round
    }

    // ---- mode: scan (and re-zero) the histogram
    int best = 0, blin = INT_MAX, bties = 0;
    for (int w = tid; w < nw4; w += nthreads) {
      // global slabs are only touched by atomics (L2) and these L1-bypassing accesses
      const uint4 v = HSMEM ? hist4[w] : __ldcg(&hist4[w]);
      if ((v.x | v.y | v.z | v.w) == 0u) continue;
      if (HSMEM) hist4[w] = make_uint4(0, 0, 0, 0); else __stcg(&hist4[w], make_uint4(0, 0, 0, 0));
      const unsigned vv[4] = {v.x, v.y, v.z, v.w};
      if (p.count16) {
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int c = (int)((vv[h >> 1] >> ((h & 1) * 16)) & 0xffffu);
          if (c > best) { best = c; blin = 8 * w + h; bties = 1; }
          else if (c == best && c > 0) ++bties;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = (int)vv[h];
          if (c > best) { best = c; blin = 4 * w + h; bties = 1; }
          else if (c == best && c > 0) ++bties;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ol = __shfl_xor_sync(0xffffffffu, blin, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bties, o);
      mode_combine(best, blin, bties, ob, ol, ot);
    }
    if (lane == 0) { red[warp] = best; red[32 + warp] = blin; red[64 + warp] = bties; }
    __syncthreads();
    if (warp == 0) {
      best = lane < nwarps ? red[lane] : 0;
      blin = lane < nwarps ? red[32 + lane] : INT_MAX;
      bties = lane < nwarps ? red[64 + lane] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ol = __shfl_xor_sync(0xffffffffu, blin, o);
        const int ot = __shfl_xor_sync(0xffffffffu, bties, o);
        mode_combine(best, blin, bties, ob, ol, ot);
      }
      if (lane == 0) {
        p.counts[rr] = best;
        p.lins[rr] = best > 0 ? blin : -1;
        p.ties[rr] = best > 0 ? bties : 0;
      }
    }
    __syncthreads();
  }

  // kernel statistics
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    st_pairs += __shfl_xor_sync(0xffffffffu, st_pairs, o);
    st_votes += __shfl_xor_sync(0xffffffffu, st_votes, o);
    st_rechecks += __shfl_xor_sync(0xffffffffu, st_rechecks, o);
  }
  if (lane == 0) {
    atomicAdd(&p.stats[0], st_pairs);
    atomicAdd(&p.stats[1], (unsigned long long)st_votes);
    atomicAdd(&p.stats[2], (unsigned long long)st_rechecks);
  }
}

size_t vote_smem_bytes(const VoteParams& p, bool hsmem, bool psmem) {
  size_t b = 0;
  if (hsmem) b += (size_t)p.hist_words * 4;
  if (psmem) b += (size_t)p.n * 16;
  b += (size_t)(p.nxt + p.nxs) * 32 + 16 * 8 + 4 * 32 * 4 + (size_t)kUnitCap * 4;
  return b;
}

cudaError_t launch_vote(const VoteParams& p, bool hsmem, bool psmem, int grid, int threads,
                        cudaStream_t stream) {
  const size_t smem = vote_smem_bytes(p, hsmem, psmem);
  cudaError_t e;
#define DSES_LAUNCH(H, PS)                                                                    \
  e = cudaFuncSetAttribute(vote_kernel<H, PS>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                           (int)smem);                                                        \
  if (e != cudaSuccess) return e;                                                             \
  vote_kernel<H, PS><<<grid, threads, smem, stream>>>(p);
  if (hsmem && psmem) { DSES_LAUNCH(true, true) }
  else if (hsmem) { DSES_LAUNCH(true, false) }
  else if (psmem) { DSES_LAUNCH(false, true) }
  else { DSES_LAUNCH(false, false) }
#undef DSES_LAUNCH
  return cudaGetLastError();
}

int vote_max_ctas_per_sm(const VoteParams& p, bool hsmem, bool psmem, int threads) {
  const size_t smem = vote_smem_bytes(p, hsmem, psmem);
  int n = 0;
  cudaError_t e;
  if (hsmem && psmem) {
    cudaFuncSetAttribute(vote_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vote_kernel<true, true>, threads, smem);
  } else if (hsmem) {
    cudaFuncSetAttribute(vote_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vote_kernel<true, false>, threads, smem);
  } else if (psmem) {
    cudaFuncSetAttribute(vote_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vote_kernel<false, true>, threads, smem);
  } else {
    cudaFuncSetAttribute(vote_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, vote_kernel<false, false>, threads, smem);
  }
  return e == cudaSuccess ? n : 0;
}

}  // namespace dses
