// Cold-start floor on this box: driver init and primary-context creation of
// an EMPTY CUDA program (compare tools/cold_start: the same plus our module).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void nop() {}
int main() {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  int n = 0;
  const auto t0 = clk::now();
  cudaGetDeviceCount(&n);
  const auto t1 = clk::now();
  cudaFree(0);
  const auto t2 = clk::now();
  nop<<<1, 1>>>();
  cudaDeviceSynchronize();
  const auto t3 = clk::now();
  std::printf("empty program: cudaGetDeviceCount %.1f ms, context (cudaFree(0)) %.1f ms, first launch %.2f ms\n",
              ms(t0, t1), ms(t1, t2), ms(t2, t3));
}
