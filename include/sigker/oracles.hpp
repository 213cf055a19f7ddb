// Independent desk-scale kernel oracles -- the reference's oracles.hpp API
// (oracles.cpp:26-383), implemented in paper_2502_20392_b200/host/oracles.cpp.
// They do not share code or formulation with the tile solver (closed forms,
// truncated signatures in the tensor algebra, a finite-difference Goursat
// solve, Picard iteration) and back the `validate` suites and the CLI
// `bench` accuracy column.  CPU, small inputs only.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "sigker/time_series.hpp"

namespace sigker::oracle {

// K of one tile with increment product rho, truncated: sum_{i<=order} rho^i / (i!)^2.
double bessel_series_kernel(double rho, int order);

// Two tiles stacked in v (x one segment, y two), increment products d11, d12:
// sum_{i+j<=2 order} d11^i d12^j / ((i+j)! i! j!).
double two_tile_closed_form(double d11, double d12, int order);

// Truncated tensor-algebra element: levels[m] holds dim^m coefficients.
struct SignatureTensor {
  std::size_t dim = 1;
  int depth = 0;
  std::vector<std::vector<double>> levels;

  static SignatureTensor identity(std::size_t dim, int depth);
  static SignatureTensor segment(std::span<const double> increment, int depth);
  void concat(const SignatureTensor& other);                 // this <- this (x) other
  void concat_segment(std::span<const double> increment);    // this <- this (x) exp(increment)
  std::size_t coefficient_count() const;
};

double signature_inner(const SignatureTensor& a, const SignatureTensor& b);
SignatureTensor path_signature(const TimeSeries& ts, int depth,
                               std::size_t memory_budget_bytes = std::size_t{1} << 30);
double truncated_signature_kernel(const TimeSeries& x, const TimeSeries& y, int depth,
                                  std::size_t memory_budget_bytes = std::size_t{1} << 30);

// The same truncation computed level by level on per-tile polynomials,
// O(rows cols depth^2) memory-light (no tensors).
double truncated_kernel_levelwise(const TimeSeries& x, const TimeSeries& y, int depth);

// Second-order finite differences on a (cols R + 1) x (rows R + 1) grid.
std::vector<double> goursat_fd_grid(const TimeSeries& x, const TimeSeries& y, int refinement);
double goursat_fd_solve(const TimeSeries& x, const TimeSeries& y, int refinement);

struct PicardResult {
  double value = 1.0;
  int iterations = 0;
  bool converged = false;
  std::vector<double> corner_history;
};
PicardResult picard_global(const TimeSeries& x, const TimeSeries& y, int refinement, int max_iterations);

}  // namespace sigker::oracle
