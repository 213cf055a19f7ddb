// Dependent-chain latency of FP64 ops and of SHFL/LDS on B200 (one warp),
// measured with clock64: informs the tile solver's ILP requirements.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, double a, double b, int iters) {
  double x = threadIdx.x * 1e-9 + 1.0;
  __shared__ double sm[64];
  sm[threadIdx.x] = x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) y = y * a;
  }
  long long t2 = clock64();
  double z = y;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31);
  }
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) idx = static_cast<int>(sm[idx & 31]) + (idx & 31);
  }
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + idx;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 4 * 8);
  const int iters = 1000;
  for (int rep = 0; rep < 2; ++rep) lat_kernel<<<1, 32>>>(out, cyc, 1.0000001, 1e-12, iters);
  long long h[4];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const double n = 16.0 * iters;
  printf("DFMA dependent latency: %.2f cycles\n", h[0] / n);
  printf("DMUL dependent latency: %.2f cycles\n", h[1] / n);
  printf("SHFL(f64) dependent latency: %.2f cycles (2 x 32-bit SHFL)\n", h[2] / n);
  printf("LDS+cvt dependent latency: %.2f cycles\n", h[3] / n);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
