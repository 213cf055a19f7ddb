// DMMA issue rate per warp: TFLOP/s of mma.sync f64 (m8n8k4 and m16n8k16)
// with W warps per SM sub-partition and C independent accumulator chains per
// warp -- how many producer warps a band needs to feed its rho (sk_sweep.cuh).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[C][2];
#pragma unroll
  for (int k = 0; k < C; ++k) c[k][0] = c[k][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < C; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

template <int C>
__global__ void k16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  double c[C][4];
#pragma unroll
  for (int k = 0; k < C; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < C; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < C; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[0] = s;
}

template <class F>
void bench(const char* name, F launch, double flops_per_warp_iter, int warps_per_smsp, int sms, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  const double warps = 4.0 * warps_per_smsp * sms;
  const double tf = flops_per_warp_iter * iters * warps / (ms * 1e-3) / 1e12;
  std::printf("%-10s %d warp(s)/SMSP: %6.2f TFLOP/s chip = %5.1f%% of 37.11\n", name, warps_per_smsp, tf,
              100 * tf / 37.11);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 2000;
  for (int w : {1, 2, 3, 4, 8}) {
    // one CTA of 4 w warps per SM: w warps on each sub-partition
    bench("884 x8", [&] { k884<8><<<sms, 128 * w>>>(out, iters); }, 8 * 512.0, w, sms, iters);
    bench("884 x16", [&] { k884<16><<<sms, 128 * w>>>(out, iters / 2); }, 16 * 512.0, w, sms, iters / 2);
    bench("16816 x4", [&] { k16816<4><<<sms, 128 * w>>>(out, iters / 4); }, 4 * 4096.0, w, sms, iters / 4);
  }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
