// Pure-math throughput of the register tile solver (no memory traffic):
// each thread chains tile_step_scaled<N> on its own series, as the sweep's
// lanes do, to bound what the sweep kernel can reach.
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2502_20392_b200/csrc/sk_device.cuh"

template <int N>
__global__ void __launch_bounds__(128) tile_loop(double* out, int iters, double d0) {
  double q[N + 1], r[N + 1], qo[N + 1], ro[N + 1];
#pragma unroll
  for (int m = 0; m <= N; ++m) {
    q[m] = (m == 0) ? 1.0 : 1e-3 * (threadIdx.x + m);
    r[m] = (m == 0) ? 1.0 : 2e-3 * m;
  }
  double delta = d0 * (1.0 + 1e-3 * threadIdx.x);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const double tot = skb::tile_step_scaled<N>(q, r, delta, qo, ro, false);
    acc += tot;
#pragma unroll
    for (int m = 0; m <= N; ++m) {
      q[m] = qo[m] * 0.5;
      r[m] = ro[m] * 0.5;
    }
    delta = -delta;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int bps : {2, 3, 4, 6, 8}) {
    const int blocks = sms * bps;
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      tile_loop<8><<<blocks, 128>>>(out, iters, 0.01);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    const double tiles = double(blocks) * 128 * iters;
    const double F = 4.0 * 81 + 2 * 8;  // algorithmic flops per tile at d = 8 (dot not executed here)
    printf("N=8 warps/SM=%d: %.3e tiles/s, F-flops %.2f TF/s (%.1f%% of 37.11)\n", bps * 4, tiles / ms * 1e3,
           tiles * (4.0 * 81) / ms / 1e9, 100.0 * tiles * (4.0 * 81) / ms / 1e9 / 37.11);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
