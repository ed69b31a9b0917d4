// dses_probe.cu -- live FP32 FFMA peak probe (the roofline denominator for the
// vote and screen kernels; MEASURED_PEAKS.json carries no FP32 figure).
#include <cuda_runtime.h>
#include "../../include/dses_b200.h"

namespace {
constexpr int kIters = 2048;

__global__ void ffma_probe(float* out, float a, float b) {
  float r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x + k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = fmaf(r[k], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int dses_probe_fp32_peak(int device, double* ffma_per_s, double* ms_out) {
  if (cudaSetDevice(device) != cudaSuccess) return DSES_E_NODEVICE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DSES_E_CUDA;
  const int threads = 512, blocks = prop.multiProcessorCount * 4;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * threads * blocks) != cudaSuccess) return DSES_E_NOMEM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    ffma_probe<<<blocks, threads>>>(out, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return DSES_E_CUDA;
  const double n = (double)blocks * threads * kIters * 16 * 8;
  if (ffma_per_s) *ffma_per_s = n / (best * 1e-3);
  if (ms_out) *ms_out = best;
  return DSES_OK;
}
