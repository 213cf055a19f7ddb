// Which hardware warp slot (%warpid; sub-partition = slot mod 4) does warp w
// of a CTA get, for CTAs of 1, 2, 4, 8 warps and several CTAs per SM?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int* out, int nwarps) {
  unsigned hw, sm;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    out[(blockIdx.x * nwarps + w) * 2] = sm;
    out[(blockIdx.x * nwarps + w) * 2 + 1] = hw;
  }
  // stay resident so later CTAs land beside earlier ones
  const long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
}
int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  int h[1 << 16];
  for (int nw : {1, 2, 4, 8}) {
    const int blocks = 148 * 4;
    probe<<<blocks, 32 * nw>>>(d, nw);
    cudaMemcpy(h, d, blocks * nw * 2 * sizeof(int), cudaMemcpyDeviceToHost);
    // SM 0's CTAs: list (block, wid -> hw slot)
    printf("%d-warp CTAs, SM 0:", nw);
    int n = 0;
    for (int b = 0; b < blocks && n < 6; ++b)
      if (h[(b * nw) * 2] == 0) {
        printf(" [blk %d:", b);
        for (int w = 0; w < nw; ++w) printf(" w%d->%d", w, h[(b * nw + w) * 2 + 1]);
        printf("]");
        ++n;
      }
    printf("\n");
  }
  return 0;
}
