// FP64 pipe microbenchmark for B200 (sm_100a): sustained DFMA rate and
// DMMA (mma.sync f64) rate. Prints TFLOP/s for each; used as the roofline
// denominator for the FP64-bound tile solver.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  double c[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int j = 0; j < 4; ++j) c[k][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int j = 0; j < 4; ++j) s += c[k][j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int tpb : {256, 512, 1024}) {
    const int iters = 20000;
    const int blocks = sms * (2048 / tpb);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, tpb>>>(out, iters, 0.999999, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA tpb=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, blocks, flops / ms / 1e9, ms);
  }
  {
    const int iters = 4000, tpb = 256, blocks = sms * 8;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dmma_m8n8k4_kernel<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (tpb / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  {
    const int iters = 1000, tpb = 256, blocks = sms * 8;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dmma_m16n8k16_kernel<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 16 * 8 * 16 * 4 * iters * (double)blocks * (tpb / 32);
    printf("DMMA m16n8k16: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  // long sustained DFMA run (~3 s) for clocks under FP64 load
  {
    const int iters = 400000, tpb = 512, blocks = sms * 4;
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, tpb>>>(out, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA sustained: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
