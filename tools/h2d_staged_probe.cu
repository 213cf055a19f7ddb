// Host->device copy of a large pageable buffer: plain pageable cudaMemcpy vs a
// staged copy (host threads memcpy chunks into two pinned staging buffers per
// thread, each chunk's DMA overlapping the next chunk's memcpy).  Input path
// of the C-ABI for pageable callers.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  const size_t n = 134217728;
  char* h = static_cast<char*>(std::malloc(n));
  std::memset(h, 1, n);
  char* d = nullptr;
  cudaMalloc(&d, n);
  cudaMemcpy(d, h, 1 << 20, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    std::printf("pageable cudaMemcpy: %.2f ms (%.1f GB/s)\n", (now() - t0) * 1e3, n / (now() - t0) / 1e9);
  }
  for (int nt : {1, 2, 4, 8, 16}) {
    for (size_t chunk : {size_t(1) << 20, size_t(4) << 20}) {
      std::vector<char*> stage(2 * nt);
      for (auto& p : stage) cudaMallocHost(&p, chunk);
      std::vector<cudaStream_t> st(nt);
      std::vector<cudaEvent_t> ev(2 * nt);
      for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        std::vector<std::thread> th;
        const size_t nchunks = (n + chunk - 1) / chunk;
        for (int t = 0; t < nt; ++t)
          th.emplace_back([&, t] {
            int k = 0;
            for (size_t c = t; c < nchunks; c += nt, ++k) {
              const int b = 2 * t + (k & 1);
              cudaEventSynchronize(ev[b]);  // the DMA that last read this buffer is done
              const size_t off = c * chunk, len = std::min(chunk, n - off);
              std::memcpy(stage[b], h + off, len);
              cudaMemcpyAsync(d + off, stage[b], len, cudaMemcpyHostToDevice, st[t]);
              cudaEventRecord(ev[b], st[t]);
            }
            cudaStreamSynchronize(st[t]);
          });
        for (auto& x : th) x.join();
        const double dt = now() - t0;
        std::printf("staged %2d threads, %zu MB chunks: %.2f ms (%.1f GB/s)\n", nt, chunk >> 20, dt * 1e3, n / dt / 1e9);
      }
      for (auto& p : stage) cudaFreeHost(p);
      for (auto& s : st) cudaStreamDestroy(s);
      for (auto& e : ev) cudaEventDestroy(e);
    }
  }
  std::printf("nproc %u\n", std::thread::hardware_concurrency());
  return 0;
}
