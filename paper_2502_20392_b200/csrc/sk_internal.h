// Internal launcher declarations shared by the C-ABI and the kernel TUs.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace skb {

struct SweepParams;

// Register-resident dot widths: d <= 16 is contracted inline in the sweep
// (dy in registers, dx streamed through L1); larger d goes through the
// skewed rho table (DP = 0).
inline int pick_dp(size_t dim) {
  if (dim <= 2) return 2;
  if (dim <= 4) return 4;
  if (dim <= 8) return 8;
  if (dim <= 16) return 16;
  return 0;
}

cudaError_t launch_increments(const double* v, size_t nseries, size_t len, size_t dim, double* out,
                              cudaStream_t st);
cudaError_t launch_max_sqnorm(const double* inc, size_t nseries, size_t count, size_t dim, double* out,
                              cudaStream_t st);
cudaError_t launch_maxrho_scan(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                               size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                               int dim, unsigned long long* out, cudaStream_t st);
cudaError_t launch_rho_table(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                             size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                             int bands, int dim, double* tab, unsigned long long tab_stride, cudaStream_t st);
cudaError_t launch_grid_init(double* grid, size_t nout, size_t lx, size_t ly, cudaStream_t st);
cudaError_t launch_step_tile_literal(double delta, int order, const double* w65, const double* in, double* out,
                                     cudaStream_t st);
cudaError_t launch_step_tile_fast(double delta, int order, const double* in, double* out, cudaStream_t st);

// Sweep instantiations: one TU per register order N in 1..16 and N = 0
// (literal arithmetic, runtime order up to 64).
cudaError_t sweep_launch(int n_template, int dp, int grid, cudaStream_t stream, const SweepParams& P);
cudaError_t sweep_occupancy(int n_template, int dp, int* blocks_per_sm);

}  // namespace skb
