// Microbenchmarks for the DSES vote-kernel design decisions on B200 (sm_100a):
// FP32 FFMA peak, shared-memory atomic throughput (ATOMS / RED.shared) with random
// spread addresses over a 138 KB histogram, and L2 (global) RED throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      r0 = fmaf(r0, a, b); r1 = fmaf(r1, a, b); r2 = fmaf(r2, a, b); r3 = fmaf(r3, a, b);
      r4 = fmaf(r4, a, b); r5 = fmaf(r5, a, b); r6 = fmaf(r6, a, b); r7 = fmaf(r7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

// 3-register FFMA form (all operands in registers, per-thread varying)
__global__ void ffma3_kernel(float* out, int iters, const float* ab) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      r0 = fmaf(r0, a, b); r1 = fmaf(r1, b, a); r2 = fmaf(r2, a, b); r3 = fmaf(r3, b, a);
      r4 = fmaf(r4, a, b); r5 = fmaf(r5, b, a); r6 = fmaf(r6, a, b); r7 = fmaf(r7, b, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

// FADD throughput (2 register operands)
__global__ void fadd_kernel(float* out, int iters, const float* ab) {
  float a = ab[threadIdx.x & 31], b = ab[32 + (threadIdx.x & 31)];
  float r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5, r6 = r0 + 6, r7 = r0 + 7;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      r0 = r0 + a; r1 = r1 - b; r2 = r2 + b; r3 = r3 - a; r4 = r4 + a; r5 = r5 - b; r6 = r6 + b; r7 = r7 - a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0 + r1 + r2 + r3 + r4 + r5 + r6 + r7;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <bool USE_RET>
__global__ void atoms_kernel(uint32_t* out, int iters, int nwords) {
  extern __shared__ uint32_t hist[];
  for (int k = threadIdx.x; k < nwords; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  uint32_t acc = 0;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      uint32_t w = (uint32_t)(((uint64_t)(s >> 8) * (uint64_t)nwords) >> 24);
      uint32_t inc = (s & 1) ? 0x10000u : 1u;
      if (USE_RET) acc += atomicAdd(&hist[w], inc);
      else atomicAdd(&hist[w], inc);
    }
  }
  __syncthreads();
  uint32_t t = 0;
  for (int k = threadIdx.x; k < nwords; k += blockDim.x) t += hist[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t + acc;
}

// same address stream, global RED into a per-CTA slab (L2 resident)
__global__ void redg_kernel(uint32_t* slabs, uint32_t* out, int iters, int nwords) {
  uint32_t* hist = slabs + (size_t)blockIdx.x * nwords;
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      uint32_t w = (uint32_t)(((uint64_t)(s >> 8) * (uint64_t)nwords) >> 24);
      atomicAdd(&hist[w], 1u);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// address generation only (cost baseline for the atomic loops)
__global__ void addr_only_kernel(uint32_t* out, int iters, int nwords) {
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x);
  uint32_t acc = 0;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      uint32_t w = (uint32_t)(((uint64_t)(s >> 8) * (uint64_t)nwords) >> 24);
      acc ^= w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s sms %d clock_attr %d MHz\n", prop.name, sms, clk_khz / 1000);
  float* fout; CK(cudaMalloc(&fout, sizeof(float) * sms * 8 * 1024));
  float* ab; CK(cudaMalloc(&ab, 64 * sizeof(float)));
  float hab[64]; for (int i = 0; i < 64; ++i) hab[i] = 0.999f + 1e-6f * i;
  CK(cudaMemcpy(ab, hab, sizeof(hab), cudaMemcpyHostToDevice));
  uint32_t* uout; CK(cudaMalloc(&uout, sizeof(uint32_t) * sms * 8 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // FFMA: grid = sms*4 blocks of 1024 threads
  {
    int iters = 4096; int blocks = sms * 4, threads = 512;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); ffma_kernel<<<blocks, threads>>>(fout, iters, 0.9999f, 0.0001f); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double ffma = (double)blocks * threads * iters * 16 * 8;
    printf("FFMA imm   : %.3f ms  %.2f TFFMA/s  (%.2f TFLOP/s)\n", ms, ffma / ms / 1e9, 2 * ffma / ms / 1e9);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); ffma3_kernel<<<blocks, threads>>>(fout, iters, ab); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("FFMA 3reg  : %.3f ms  %.2f TFFMA/s  (%.2f TFLOP/s)\n", ms, ffma / ms / 1e9, 2 * ffma / ms / 1e9);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); fadd_kernel<<<blocks, threads>>>(fout, iters, ab); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("FADD 2reg  : %.3f ms  %.2f Tops/s\n", ms, ffma / ms / 1e9);
  }
  // shared atomics: 1 CTA/SM, 1024 threads, 34461 words (68921 16-bit bins)
  const int nwords_list[3] = {34461, 4096, 256};
  CK(cudaFuncSetAttribute(atoms_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(atoms_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int t = 0; t < 3; ++t) {
    int nwords = nwords_list[t];
    for (int threads : {256, 512, 1024}) {
      int iters = 2048; int blocks = sms;
      double n = (double)blocks * threads * iters * 8;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); atoms_kernel<true><<<blocks, threads, nwords * 4>>>(uout, iters, nwords); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      double rate_ret = n / ms / 1e6;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); atoms_kernel<false><<<blocks, threads, nwords * 4>>>(uout, iters, nwords); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      double rate_red = n / ms / 1e6;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); addr_only_kernel<<<blocks, threads>>>(uout, iters, nwords); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      double rate_addr = n / ms / 1e6;
      printf("ATOMS words=%6d thr=%4d: ret %.1f G/s  noret %.1f G/s  addr-only %.1f G/s  (per SM per clk@1.9GHz: %.3f / %.3f)\n",
             nwords, threads, rate_ret / 1e3, rate_red / 1e3, rate_addr / 1e3,
             rate_ret / 1e3 / sms / 1.9, rate_red / 1e3 / sms / 1.9);
    }
  }
  // 2 CTAs per SM with half-size histograms
  {
    int nwords = 17231, threads = 512, iters = 2048, blocks = sms * 2;
    double n = (double)blocks * threads * iters * 8;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); atoms_kernel<false><<<blocks, threads, nwords * 4>>>(uout, iters, nwords); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("ATOMS 2CTA/SM words=%d: noret %.1f G/s\n", nwords, n / ms / 1e9);
  }
  // global RED into per-CTA L2 slabs
  {
    int nwords = 68921; int threads = 1024, iters = 512;
    for (int blocks : {sms, sms * 2}) {
      uint32_t* slabs; CK(cudaMalloc(&slabs, (size_t)blocks * nwords * 4)); cudaMemset(slabs, 0, (size_t)blocks * nwords * 4);
      double n = (double)blocks * threads * iters * 8;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0); redg_kernel<<<blocks, threads>>>(slabs, uout, iters, nwords); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("REDG blocks=%d words=%d: %.1f G/s\n", blocks, nwords, n / ms / 1e9);
      cudaFree(slabs);
    }
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
