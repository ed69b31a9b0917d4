// dses_sweep.cu -- dense translation sweep of the mode-optimality check.
//
// Replaces _kernels.sweep_inlier_best (_kernels.py:384-410), the brute-force
// side of harness.run_oracle_checks (harness.py:418-446): for every
// translation t of the lattice t0 x t1 x t2, count the sources i that have
// some difference c_ij = y_j - R x_i inside the open Chebyshev ball
// |c_ij - t|_inf < half, and return the maximum count.
//
// B200 layout: one thread per lattice translation (the innermost axis t2 on
// consecutive lanes), grid-stride over the lattice with the grid sized to
// the SM count; the n*m differences are staged once per CTA in shared
// memory and read at warp-uniform addresses (broadcast).  Comparisons are
// binary64 subtractions and compares, exactly the reference's, so the count
// is bit-identical; the maximum is a warp max + one atomicMax per warp.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dses_b200.h"

namespace dses {

int api_fail(int code, const char* what);  // dses_capi.cu: sets dses_last_error()
constexpr int kSweepThreads = 256;

template <bool SMEM>
__global__ void __launch_bounds__(kSweepThreads) sweep_inlier_kernel(
    const double* __restrict__ cands, int n, int m, double half, const double* __restrict__ t0,
    const double* __restrict__ t1, const double* __restrict__ t2, int64_t n1, int64_t n2,
    int64_t total, int* best) {
  extern __shared__ double sc[];
  const double* c = cands;
  if (SMEM) {
    for (int k = threadIdx.x; k < 3 * n * m; k += blockDim.x) sc[k] = cands[k];
    __syncthreads();
    c = sc;
  }
  int local = 0;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx / (n1 * n2), rem = idx - a * (n1 * n2);
    const int64_t b = rem / n2, cc = rem - b * n2;
    const double ta = t0[a], tb = t1[b], tc = t2[cc];
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
      const double* row = c + (size_t)3 * i * m;
      for (int j = 0; j < m; ++j) {
        if (fabs(__dsub_rn(row[3 * j], ta)) < half && fabs(__dsub_rn(row[3 * j + 1], tb)) < half &&
            fabs(__dsub_rn(row[3 * j + 2], tc)) < half) {
          ++cnt;
          break;
        }
      }
    }
    local = max(local, cnt);
  }
  for (int o = 16; o; o >>= 1) local = max(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0 && local > 0) atomicMax(best, local);
}

}  // namespace dses

// Host pointers in, host scalar out (the reference kernel's calling
// convention: cands (n*m, 3) row-major by source, three axis arrays).
extern "C" int dses_sweep_inlier_best(int device, const double* cands, int64_t n, int64_t m,
                                      double half, const double* t0, int64_t n0, const double* t1,
                                      int64_t n1, const double* t2, int64_t n2, int64_t* best_out) {
  if (!best_out || n < 0 || m < 0 || n0 < 0 || n1 < 0 || n2 < 0)
    return dses::api_fail(DSES_E_INVALID, "negative size or null output");
  if (n > INT32_MAX / 3 || m > INT32_MAX / 3 || n * m > INT32_MAX / 3)
    return dses::api_fail(DSES_E_INVALID, "n*m too large");
  *best_out = 0;
  const int64_t total = n0 * n1 * n2;
  if (total == 0 || n == 0 || m == 0) return DSES_OK;
  if (!cands || !t0 || !t1 || !t2)
    return dses::api_fail(DSES_E_INVALID, "null input");
  if (cudaSetDevice(device) != cudaSuccess)
    return dses::api_fail(DSES_E_NODEVICE, "no usable CUDA device");
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return dses::api_fail(DSES_E_CUDA, "device query failed");
  const size_t cb = sizeof(double) * 3 * (size_t)(n * m);
  const size_t ab = sizeof(double) * (size_t)(n0 + n1 + n2);
  char* buf = nullptr;
  if (cudaMalloc(&buf, cb + ab + 16) != cudaSuccess)
    return dses::api_fail(DSES_E_NOMEM, "device allocation failed");
  double* dc = reinterpret_cast<double*>(buf);
  double* d0 = dc + 3 * n * m;
  double* d1 = d0 + n0;
  double* d2 = d1 + n1;
  int* dbest = reinterpret_cast<int*>(d2 + n2);
  cudaError_t e = cudaMemcpy(dc, cands, cb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d0, t0, sizeof(double) * n0, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d1, t1, sizeof(double) * n1, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d2, t2, sizeof(double) * n2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dbest, 0, sizeof(int));
  if (e == cudaSuccess) {
    const int64_t want = (total + dses::kSweepThreads - 1) / dses::kSweepThreads;
    const int grid = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
    if (cb <= 48 * 1024)
      dses::sweep_inlier_kernel<true><<<grid, dses::kSweepThreads, cb>>>(
          dc, (int)n, (int)m, half, d0, d1, d2, n1, n2, total, dbest);
    else
      dses::sweep_inlier_kernel<false><<<grid, dses::kSweepThreads>>>(
          dc, (int)n, (int)m, half, d0, d1, d2, n1, n2, total, dbest);
    e = cudaGetLastError();
  }
  int best = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&best, dbest, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return dses::api_fail(DSES_E_CUDA, cudaGetErrorString(e));
  *best_out = best;
  return DSES_OK;
}
