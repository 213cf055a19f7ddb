// Dispatch from a runtime order to the per-order sweep instantiations
// (sk_sweep_inst.cu compiled once per SK_N).
#include <cuda_runtime.h>

#include "sk_internal.h"
#include "sk_sweep.cuh"

namespace skb {

cudaError_t sweep_launch_n0(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n0(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n1(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n1(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n2(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n2(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n3(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n3(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n4(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n4(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n5(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n5(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n6(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n6(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n7(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n7(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n8(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n8(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n9(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n9(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n10(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n10(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n11(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n11(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n12(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n12(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n13(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n13(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n14(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n14(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n15(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n15(int dp, int* blocks_per_sm);
cudaError_t sweep_launch_n16(int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy_n16(int dp, int* blocks_per_sm);

cudaError_t sweep_launch(int n_template, int dp, int grid, cudaStream_t stream, const SweepParams& P) {
  switch (n_template) {
    case 0: return sweep_launch_n0(dp, grid, stream, P);
    case 1: return sweep_launch_n1(dp, grid, stream, P);
    case 2: return sweep_launch_n2(dp, grid, stream, P);
    case 3: return sweep_launch_n3(dp, grid, stream, P);
    case 4: return sweep_launch_n4(dp, grid, stream, P);
    case 5: return sweep_launch_n5(dp, grid, stream, P);
    case 6: return sweep_launch_n6(dp, grid, stream, P);
    case 7: return sweep_launch_n7(dp, grid, stream, P);
    case 8: return sweep_launch_n8(dp, grid, stream, P);
    case 9: return sweep_launch_n9(dp, grid, stream, P);
    case 10: return sweep_launch_n10(dp, grid, stream, P);
    case 11: return sweep_launch_n11(dp, grid, stream, P);
    case 12: return sweep_launch_n12(dp, grid, stream, P);
    case 13: return sweep_launch_n13(dp, grid, stream, P);
    case 14: return sweep_launch_n14(dp, grid, stream, P);
    case 15: return sweep_launch_n15(dp, grid, stream, P);
    case 16: return sweep_launch_n16(dp, grid, stream, P);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t sweep_occupancy(int n_template, int dp, int* blocks_per_sm) {
  switch (n_template) {
    case 0: return sweep_occupancy_n0(dp, blocks_per_sm);
    case 1: return sweep_occupancy_n1(dp, blocks_per_sm);
    case 2: return sweep_occupancy_n2(dp, blocks_per_sm);
    case 3: return sweep_occupancy_n3(dp, blocks_per_sm);
    case 4: return sweep_occupancy_n4(dp, blocks_per_sm);
    case 5: return sweep_occupancy_n5(dp, blocks_per_sm);
    case 6: return sweep_occupancy_n6(dp, blocks_per_sm);
    case 7: return sweep_occupancy_n7(dp, blocks_per_sm);
    case 8: return sweep_occupancy_n8(dp, blocks_per_sm);
    case 9: return sweep_occupancy_n9(dp, blocks_per_sm);
    case 10: return sweep_occupancy_n10(dp, blocks_per_sm);
    case 11: return sweep_occupancy_n11(dp, blocks_per_sm);
    case 12: return sweep_occupancy_n12(dp, blocks_per_sm);
    case 13: return sweep_occupancy_n13(dp, blocks_per_sm);
    case 14: return sweep_occupancy_n14(dp, blocks_per_sm);
    case 15: return sweep_occupancy_n15(dp, blocks_per_sm);
    case 16: return sweep_occupancy_n16(dp, blocks_per_sm);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace skb
