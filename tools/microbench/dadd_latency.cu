// Dependent binary64 add chain latency (one thread): cycles per DADD.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dadd tools/microbench/dadd_latency.cu && /tmp/dadd
#include <cstdio>
__global__ void chain(const double* v, int n, double* out, long long* cyc) {
  double acc = 0.0;
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, v[i & 255]);
  const long long t1 = clock64();
  *out = acc;
  *cyc = t1 - t0;
}
int main() {
  double *v, *o;
  long long* c;
  cudaMalloc(&v, 256 * 8);
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1.0 / (i + 3);
  cudaMemcpy(v, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    chain<<<1, 1>>>(v, 100000, o, c);
    long long cy;
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("%.2f cycles per dependent DADD\n", cy / 100000.0);
  }
  return 0;
}
