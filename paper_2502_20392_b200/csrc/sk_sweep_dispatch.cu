// Dispatch from a runtime order to the per-order sweep instantiations
// (sk_sweep_inst.cu compiled once per SK_N; weak so that experimental builds
// with a subset of orders still link).
#include <cuda_runtime.h>

#include "sk_internal.h"
#include "sk_sweep.cuh"

namespace skb {

__attribute__((weak)) cudaError_t sweep_launch_n0(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n0(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n1(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n1(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n2(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n2(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n3(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n3(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n4(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n4(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n5(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n5(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n6(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n6(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n7(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n7(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n8(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n8(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n9(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n9(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n10(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n10(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n11(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n11(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n12(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n12(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n13(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n13(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n14(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n14(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n15(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n15(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);
__attribute__((weak)) cudaError_t sweep_launch_n16(int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream, const SweepParams& P);
__attribute__((weak)) cudaError_t sweep_occupancy_n16(int dp, bool exact, bool extras, bool paired, int* blocks_per_sm);

cudaError_t sweep_launch(int n_template, int dp, bool exact, bool extras, bool paired, int grid, cudaStream_t stream,
                         const SweepParams& P) {
  switch (n_template) {
    case 0: return sweep_launch_n0 ? sweep_launch_n0(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 1: return sweep_launch_n1 ? sweep_launch_n1(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 2: return sweep_launch_n2 ? sweep_launch_n2(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 3: return sweep_launch_n3 ? sweep_launch_n3(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 4: return sweep_launch_n4 ? sweep_launch_n4(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 5: return sweep_launch_n5 ? sweep_launch_n5(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 6: return sweep_launch_n6 ? sweep_launch_n6(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 7: return sweep_launch_n7 ? sweep_launch_n7(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 8: return sweep_launch_n8 ? sweep_launch_n8(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 9: return sweep_launch_n9 ? sweep_launch_n9(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 10: return sweep_launch_n10 ? sweep_launch_n10(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 11: return sweep_launch_n11 ? sweep_launch_n11(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 12: return sweep_launch_n12 ? sweep_launch_n12(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 13: return sweep_launch_n13 ? sweep_launch_n13(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 14: return sweep_launch_n14 ? sweep_launch_n14(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 15: return sweep_launch_n15 ? sweep_launch_n15(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    case 16: return sweep_launch_n16 ? sweep_launch_n16(dp, exact, extras, paired, grid, stream, P) : cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t sweep_occupancy(int n_template, int dp, bool exact, bool extras, bool paired, int* blocks_per_sm) {
  switch (n_template) {
    case 0: return sweep_occupancy_n0 ? sweep_occupancy_n0(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 1: return sweep_occupancy_n1 ? sweep_occupancy_n1(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 2: return sweep_occupancy_n2 ? sweep_occupancy_n2(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 3: return sweep_occupancy_n3 ? sweep_occupancy_n3(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 4: return sweep_occupancy_n4 ? sweep_occupancy_n4(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 5: return sweep_occupancy_n5 ? sweep_occupancy_n5(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 6: return sweep_occupancy_n6 ? sweep_occupancy_n6(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 7: return sweep_occupancy_n7 ? sweep_occupancy_n7(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 8: return sweep_occupancy_n8 ? sweep_occupancy_n8(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 9: return sweep_occupancy_n9 ? sweep_occupancy_n9(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 10: return sweep_occupancy_n10 ? sweep_occupancy_n10(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 11: return sweep_occupancy_n11 ? sweep_occupancy_n11(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 12: return sweep_occupancy_n12 ? sweep_occupancy_n12(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 13: return sweep_occupancy_n13 ? sweep_occupancy_n13(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 14: return sweep_occupancy_n14 ? sweep_occupancy_n14(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 15: return sweep_occupancy_n15 ? sweep_occupancy_n15(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    case 16: return sweep_occupancy_n16 ? sweep_occupancy_n16(dp, exact, extras, paired, blocks_per_sm) : cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace skb
