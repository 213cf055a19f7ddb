// sigker/tile_series.hpp -- single-tile algebra of the drop-in C++ API
// (reference tile_series.hpp:8-114).  These are the unfused specification
// functions; they run on the host (cheap, O(N^2) per call).  The hot path
// (the fused sweep) lives on the GPU behind wavefront.hpp.
#pragma once

#include <cstddef>
#include <iosfwd>
#include <span>
#include <vector>

namespace sigker::tile {

inline constexpr int kMaxOrder = 64;

// Coefficients c[i][j] of sum_{i,j<=N} c[i][j] u^i v^j, row-major in i.
struct CoeffMatrix {
  int order = 0;
  std::vector<double> entries;
  double at(int i, int j) const { return entries[static_cast<std::size_t>(i) * (order + 1) + j]; }
  double& at(int i, int j) { return entries[static_cast<std::size_t>(i) * (order + 1) + j]; }
};

enum class BoundaryAxis { AlongU, AlongV };

// A series along one tile edge (N+1 coefficients).
struct BoundarySeries {
  BoundaryAxis axis = BoundaryAxis::AlongU;
  std::vector<double> a;
  static BoundarySeries unit(BoundaryAxis axis, int order);
};

std::vector<double> power_vector(double x, int order);
CoeffMatrix build_W(int order);
CoeffMatrix build_A(double delta, int order);
CoeffMatrix build_B(const BoundarySeries& alpha, const BoundarySeries& beta, int order);
CoeffMatrix tile_coeffs(double delta, const BoundarySeries& alpha, const BoundarySeries& beta, int order);
double eval_series(const CoeffMatrix& c, double u, double v);
BoundarySeries top_boundary(const CoeffMatrix& c);
BoundarySeries right_boundary(const CoeffMatrix& c);
CoeffMatrix neumann_coeffs_slow(double delta, const BoundarySeries& alpha, const BoundarySeries& beta, int order,
                                int iters);
double monomial_propagation(double delta, int power, int n);
void dump_csv(const CoeffMatrix& c, std::ostream& out);

namespace detail {
std::span<const double> factorials();
void build_W_into(std::span<double> w, int order);
void build_A_into(std::span<double> a, double delta, int order);
void check_corner(double alpha0, double beta0);
// negative-control hook: also flips W[1][1] inside the GPU sweep
void set_w_fault_for_testing(bool enabled);
bool w_fault_for_testing();
}  // namespace detail

}  // namespace sigker::tile
