// One translation unit per truncation order: compiled once per SK_N value
// (Makefile) so the 17 x 5 sweep instantiations build in parallel.
#include <cuda_runtime.h>

#include "sk_sweep.cuh"

#ifndef SK_N
#error "SK_N must be defined"
#endif

namespace skb {

template <int N, int DP>
static cudaError_t launch_one(int grid, cudaStream_t stream, const SweepParams& P) {
  const size_t smem = static_cast<size_t>(kSweepWarps) * stage_doubles_per_warp<N>() * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<N, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  sweep_kernel<N, DP><<<grid, kSweepWarps * 32, smem, stream>>>(P);
  return cudaGetLastError();
}

template <int N, int DP>
static cudaError_t occupancy_one(int* blocks_per_sm) {
  const size_t smem = static_cast<size_t>(kSweepWarps) * stage_doubles_per_warp<N>() * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(sweep_kernel<N, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sweep_kernel<N, DP>, kSweepWarps * 32, smem);
}

#define SK_CAT2(a, b) a##b
#define SK_CAT(a, b) SK_CAT2(a, b)

cudaError_t SK_CAT(sweep_launch_n, SK_N)(int dp, int grid, cudaStream_t stream, const SweepParams& P) {
  switch (dp) {
    case 0: return launch_one<SK_N, 0>(grid, stream, P);
    case 2: return launch_one<SK_N, 2>(grid, stream, P);
    case 4: return launch_one<SK_N, 4>(grid, stream, P);
    case 8: return launch_one<SK_N, 8>(grid, stream, P);
    case 16: return launch_one<SK_N, 16>(grid, stream, P);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t SK_CAT(sweep_occupancy_n, SK_N)(int dp, int* blocks_per_sm) {
  switch (dp) {
    case 0: return occupancy_one<SK_N, 0>(blocks_per_sm);
    case 2: return occupancy_one<SK_N, 2>(blocks_per_sm);
    case 4: return occupancy_one<SK_N, 4>(blocks_per_sm);
    case 8: return occupancy_one<SK_N, 8>(blocks_per_sm);
    case 16: return occupancy_one<SK_N, 16>(blocks_per_sm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace skb
