// Host->device copy of a large pageable buffer: plain pageable cudaMemcpy vs
// registering the pages first (cudaHostRegister) -- input path of the C-ABI.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t n = 134217728;
  char* h = static_cast<char*>(std::malloc(n));
  std::memset(h, 1, n);
  void* d = nullptr;
  cudaMalloc(&d, n);
  cudaMemcpy(d, h, 1 << 20, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    double t1 = now();
    cudaHostRegister(h, n, cudaHostRegisterDefault);
    double t2 = now();
    cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    double t3 = now();
    cudaHostUnregister(h);
    double t4 = now();
    std::printf("pageable %.2f ms | register %.2f + copy %.2f + unregister %.2f ms\n", 1e3 * (t1 - t0),
                1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3));
  }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
