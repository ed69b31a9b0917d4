// dses_sparse.cu -- the histogram mode for translation lattices too large for
// a dense histogram (shared memory or per-CTA global slabs).
//
// Replaces _kernels.mode_sparse_batch / _mode_sparse_one (_kernels.py:196-294):
// per rotation, every pair (i, j) with an in-window binary64 bin (reference
// operation order) emits the key lin * N + i (int64; dedup = unique keys);
// keys are radix-sorted, deduplicated, run-length encoded by lin, and the
// mode is the longest run (ties: smallest lin, which comes first in sorted
// order; `ties` = runs of that length).  Same (count, lin, ties) as the dense
// path and as the reference (TestDenseSparseAgreement, reference
// tests/test_mode_search.py:270-293).
//
// Used for mode queries (dses_mode_batch / dses_mode_grid, hence
// mode_translation without bounds at fine bins) when the lattice exceeds
// kDenseMaxBins; the work per rotation is N*M exact binary64 pairs plus a
// sort, i.e. the reference's own sparse algorithm on the GPU.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <climits>
#include "dses_common.cuh"

namespace dses {


// Keys of one rotation: lin * n + i for in-window pairs, compacted.
__global__ void sparse_keys_kernel(SparseParams s, int64_t r, unsigned long long* keys,
                                   unsigned long long* nkeys) {
  __shared__ double R[9];
  if (threadIdx.x < 9) R[threadIdx.x] = rotation_entry(s.rot, r, threadIdx.x);
  __syncthreads();
  const int64_t total = (int64_t)s.n * s.m;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < total;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = base + threadIdx.x;
    bool ok = false;
    unsigned long long key = 0;
    if (e < total) {
      const int i = (int)(e / s.m), j = (int)(e % s.m);
      const double x0 = s.x[3 * i], x1 = s.x[3 * i + 1], x2 = s.x[3 * i + 2];
      const double p0 = rot_row(R, 0, x0, x1, x2);
      const double p1 = rot_row(R, 1, x0, x1, x2);
      const double p2 = rot_row(R, 2, x0, x1, x2);
      const double* yj = s.y + 3 * j;
      // _kernels.py:244-253 (binary64, reference operation order)
      const double q0 = dmul(dsub(yj[0], p0), s.inv_bin);
      const double f0 = dsub(copysign(floor(dadd(fabs(q0), 0.5)), q0), s.flo0);
      const double q1 = dmul(dsub(yj[1], p1), s.inv_bin);
      const double f1 = dsub(copysign(floor(dadd(fabs(q1), 0.5)), q1), s.flo1);
      const double q2 = dmul(dsub(yj[2], p2), s.inv_bin);
      const double f2 = dsub(copysign(floor(dadd(fabs(q2), 0.5)), q2), s.flo2);
      ok = (f0 >= 0.0) & (f0 < s.fd0) & (f1 >= 0.0) & (f1 < s.fd1) & (f2 >= 0.0) & (f2 < s.fd2);
      if (ok) {
        const int64_t lin = ((int64_t)f0 * s.d1 + (int64_t)f1) * s.d2 + (int64_t)f2;
        key = (unsigned long long)(lin * s.n + i);
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if (m) {
      unsigned long long slot = 0;
      if (lane == 0) slot = atomicAdd(nkeys, (unsigned long long)__popc(m));
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (ok) keys[slot + __popc(m & ((1u << lane) - 1u))] = key;
    }
  }
}

__global__ void keys_to_lins_kernel(const unsigned long long* ukeys, int64_t count, int n,
                                    unsigned long long* lins) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    lins[k] = ukeys[k] / (unsigned long long)n;
}

// One block: longest run (first = smallest lin on ties) and the number of
// runs of that length.  Writes count / lin / ties of rotation slot rr.
__global__ void sparse_mode_kernel(const unsigned long long* run_lins, const int* run_len,
                                   const int* nruns, int64_t rr, int* counts, long long* lins,
                                   int* ties) {
  __shared__ int sbest[32], sidx[32], sties[32];
  const int nr = *nruns;
  int best = 0, bidx = INT_MAX, bt = 0;
  for (int k = threadIdx.x; k < nr; k += blockDim.x) {
    const int c = run_len[k];
    if (c > best) { best = c; bidx = k; bt = 1; }
    else if (c == best && c > 0) { bidx = min(bidx, k); ++bt; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (ob > best) { best = ob; bidx = oi; bt = ot; }
    else if (ob == best) { bidx = min(bidx, oi); bt += ot; }
  }
  if (lane == 0) { sbest[warp] = best; sidx[warp] = bidx; sties[warp] = bt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    best = 0; bidx = INT_MAX; bt = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (sbest[w] > best) { best = sbest[w]; bidx = sidx[w]; bt = sties[w]; }
      else if (sbest[w] == best) { bidx = min(bidx, sidx[w]); bt += sties[w]; }
    }
    counts[rr] = best;
    lins[rr] = best > 0 ? (long long)run_lins[bidx] : -1;
    ties[rr] = best > 0 ? bt : 0;
  }
}

// Scratch for one rotation's keys: 2 key arrays (sort double buffer), lins,
// run outputs and CUB temp storage, all carved from `scratch` (bytes given by
// sparse_scratch_bytes).
size_t sparse_scratch_bytes(int64_t n, int64_t m) {
  const size_t k = (size_t)(n * m);
  size_t temp = 0, t2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, temp, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int64_t)k);
  cub::DeviceSelect::Unique(nullptr, t2, (const unsigned long long*)nullptr,
                            (unsigned long long*)nullptr, (int*)nullptr, (int64_t)k);
  temp = std::max(temp, t2);
  cub::DeviceRunLengthEncode::Encode(nullptr, t2, (const unsigned long long*)nullptr,
                                     (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr,
                                     (int64_t)k);
  temp = std::max(temp, t2);
  return 4 * k * 8 + k * 4 + 64 + temp + 8 * 256;
}

cudaError_t launch_sparse_modes(const SparseParams& s, int64_t r_begin, int64_t r_count,
                                void* scratch, size_t scratch_bytes, unsigned long long* counters,
                                int* counts, long long* lins, int* ties, int sms,
                                cudaStream_t st) {
  const size_t k = (size_t)((int64_t)s.n * s.m);
  auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
  unsigned char* base = static_cast<unsigned char*>(scratch);
  size_t off = 0;
  auto* keys = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* sorted = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* ukeys = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* ulins = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* runlen = reinterpret_cast<int*>(base + off); off = align(off + k * 4);
  int* nunique = reinterpret_cast<int*>(base + off); off = align(off + 16);
  int* nruns = nunique + 1;
  void* temp = base + off;
  const size_t temp_bytes = scratch_bytes > off ? scratch_bytes - off : 0;
  cudaError_t e = cudaSuccess;
  for (int64_t rr = 0; rr < r_count; ++rr) {
    e = cudaMemsetAsync(counters, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const int blocks = (int)std::min<int64_t>((int64_t)sms * 8, ((int64_t)k + 255) / 256);
    sparse_keys_kernel<<<std::max(blocks, 1), 256, 0, st>>>(s, r_begin + rr, keys, counters);
    unsigned long long nk = 0;
    e = cudaMemcpyAsync(&nk, counters, sizeof nk, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (nk == 0) {
      const int zero = 0;
      const long long neg = -1;
      cudaMemcpyAsync(counts + rr, &zero, sizeof zero, cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(lins + rr, &neg, sizeof neg, cudaMemcpyHostToDevice, st);
      e = cudaMemcpyAsync(ties + rr, &zero, sizeof zero, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return e;
      e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return e;
      continue;
    }
    size_t tb = temp_bytes;
    e = cub::DeviceRadixSort::SortKeys(temp, tb, keys, sorted, (int64_t)nk, 0, 64, st);
    if (e != cudaSuccess) return e;
    tb = temp_bytes;
    e = cub::DeviceSelect::Unique(temp, tb, sorted, ukeys, nunique, (int64_t)nk, st);
    if (e != cudaSuccess) return e;
    int nu = 0;
    e = cudaMemcpyAsync(&nu, nunique, sizeof nu, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    keys_to_lins_kernel<<<std::max(1, std::min(sms * 8, (nu + 255) / 256)), 256, 0, st>>>(
        ukeys, nu, s.n, ulins);
    // runs over the (sorted) unique lins; RLE writes the run lins into `sorted`
    tb = temp_bytes;
    e = cub::DeviceRunLengthEncode::Encode(temp, tb, ulins, sorted, runlen, nruns, (int64_t)nu, st);
    if (e != cudaSuccess) return e;
    sparse_mode_kernel<<<1, 1024, 0, st>>>(sorted, runlen, nruns, rr, counts, lins, ties);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Flat bins of a sort-based mode batch narrowed to the int32 the search's
// select / score stages read (the lattice is < 2^31 bins there).
__global__ void narrow_lins_kernel(const long long* __restrict__ in, int* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int)in[i];
}

cudaError_t launch_narrow_lins(const long long* in, int* out, int64_t n, int sms, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 4, (n + 255) / 256));
  narrow_lins_kernel<<<blocks, 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

// The full vote map of one rotation (mode_search.translation_histogram,
// mode_search.py:205-235): keys of rotation 0 of `s.rot` sorted, deduplicated
// per (bin, source) when `dedup`, run-length encoded by bin.  Outputs live in
// the scratch: *out_lins (ascending flat bins, u64), *out_counts (int32) and
// *out_n (device int, number of bins); *nkeys_host = pairs in the lattice.
cudaError_t launch_sparse_histogram(const SparseParams& s, bool dedup, void* scratch,
                                    size_t scratch_bytes, unsigned long long* counter,
                                    unsigned long long** out_lins, int** out_counts, int** out_n,
                                    unsigned long long* nkeys_host, int sms, cudaStream_t st) {
  const size_t k = (size_t)((int64_t)s.n * s.m);
  auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
  unsigned char* base = static_cast<unsigned char*>(scratch);
  size_t off = 0;
  auto* keys = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* sorted = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* ukeys = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* ulins = reinterpret_cast<unsigned long long*>(base + off); off = align(off + k * 8);
  auto* runlen = reinterpret_cast<int*>(base + off); off = align(off + k * 4);
  int* nunique = reinterpret_cast<int*>(base + off); off = align(off + 16);
  int* nruns = nunique + 1;
  void* temp = base + off;
  const size_t temp_bytes = scratch_bytes > off ? scratch_bytes - off : 0;
  *out_lins = keys;  // free once the keys are sorted
  *out_counts = runlen;
  *out_n = nruns;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(nruns, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int blocks = (int)std::min<int64_t>((int64_t)sms * 8, ((int64_t)k + 255) / 256);
  sparse_keys_kernel<<<std::max(blocks, 1), 256, 0, st>>>(s, 0, keys, counter);
  unsigned long long nk = 0;
  e = cudaMemcpyAsync(&nk, counter, sizeof nk, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  *nkeys_host = nk;
  if (nk == 0) return cudaSuccess;
  size_t tb = temp_bytes;
  e = cub::DeviceRadixSort::SortKeys(temp, tb, keys, sorted, (int64_t)nk, 0, 64, st);
  if (e != cudaSuccess) return e;
  const unsigned long long* src = sorted;
  int64_t count = (int64_t)nk;
  if (dedup) {
    tb = temp_bytes;
    e = cub::DeviceSelect::Unique(temp, tb, sorted, ukeys, nunique, (int64_t)nk, st);
    if (e != cudaSuccess) return e;
    int nu = 0;
    e = cudaMemcpyAsync(&nu, nunique, sizeof nu, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    src = ukeys;
    count = nu;
  }
  keys_to_lins_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, (count + 255) / 256)),
                        256, 0, st>>>(src, count, s.n, ulins);
  tb = temp_bytes;
  e = cub::DeviceRunLengthEncode::Encode(temp, tb, ulins, keys, runlen, nruns, count, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace dses
