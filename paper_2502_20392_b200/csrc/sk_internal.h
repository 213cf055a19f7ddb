// Internal launcher declarations shared by the C-ABI and the kernel TUs.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace skb {

struct SweepParams;

// Register-resident dot widths: d <= 16 is contracted inline in the sweep
// (dy in registers, dx streamed through shared memory); larger d (DP = 0) is
// contracted by the band CTA's producer warp on the FP64 tensor cores.
inline int pick_dp(size_t dim) {
  if (dim <= 2) return 2;
  if (dim <= 4) return 4;
  if (dim <= 8) return 8;
  if (dim <= 16) return 16;
  return 0;
}

// Device increment layout: per series `len` rows of `ld` doubles, row 0 zero,
// row k+1 = dz_k zero-padded to ld (ld = pick_dp(d), or d rounded up to a
// multiple of 4 on the table path: 16-byte rows, whole DMMA k-steps).
inline size_t inc_ld(size_t dim) {
  const int dp = pick_dp(dim);
  return dp > 0 ? static_cast<size_t>(dp) : (dim + 3) / 4 * 4;
}
// Increments rows (zero row first, ld doubles per row); with sqn (device,
// nseries doubles) also each series' max squared increment norm, fused for
// ld <= 16.
cudaError_t launch_increments(const double* v, size_t nseries, size_t len, size_t dim, size_t ld, double* out,
                              cudaStream_t st, double* sqn = nullptr);
cudaError_t launch_max_sqnorm(const double* inc, size_t nseries, size_t count, size_t dim, size_t ld, double* out,
                              cudaStream_t st);
cudaError_t launch_maxrho_scan(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                               size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                               int dim, int ld, unsigned long long* out, cudaStream_t st);
// rho[i][j] tables (rows x cols, row-major) for the large-d path when they
// fit the memory budget: DMMA GEMM, or the bit-exact sequential dot when `exact`.
// rowdone (DMMA only, optional): npairs x ceil(rows / 64) counters, each
// counting the 64 x 64 tiles of its row block written (ceil(cols / 64) when done).
cudaError_t launch_rho_table(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                             size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                             int dim, int ld, bool exact, double* tab, unsigned long long tab_stride,
                             cudaStream_t st, unsigned* rowdone = nullptr);
cudaError_t launch_reset_slots(const uint32_t* idx, size_t n, unsigned long long* err, cudaStream_t st);
cudaError_t launch_gather_slots(const uint32_t* idx, size_t n, const double* values, const unsigned long long* err,
                                unsigned long long* out, cudaStream_t st);
cudaError_t launch_scatter_gram(const uint32_t* pi, const uint32_t* pj, size_t n, size_t m, const double* values,
                                const unsigned long long* err, double* mat, cudaStream_t st);
cudaError_t launch_grid_init(double* grid, size_t nout, size_t lx, size_t ly, cudaStream_t st);
cudaError_t launch_step_tile_literal(double delta, int order, const double* w65, const double* in, double* out,
                                     cudaStream_t st);
cudaError_t launch_step_tile_fast(double delta, int order, const double* in, double* out, cudaStream_t st);

// Sweep instantiations: one TU per register order N in 1..16 and N = 0
// (literal arithmetic, runtime order up to 64).
// exact: reference-identical delta (sequential non-FMA dot) + per-pair
// max|delta| tracking; otherwise an FMA dot and no max tracking.
// extras: knot grid / diagonal outputs.
// literal: the reference's arithmetic at this compile-time order (registers;
// n_template 8 only) -- strict-corner re-sweeps.
cudaError_t sweep_launch(int n_template, int dp, bool exact, bool extras, bool literal, int grid, cudaStream_t stream,
                         const SweepParams& P);
cudaError_t sweep_occupancy(int n_template, int dp, bool exact, bool extras, bool literal, int* blocks_per_sm);

}  // namespace skb
