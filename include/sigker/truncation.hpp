// sigker/truncation.hpp -- truncation-order policy of the drop-in C++ API
// (reference truncation.hpp:10-51).
#pragma once

#include <cstddef>

namespace sigker {

struct TruncationPolicy {
  enum class Mode { kFixed, kAdaptive };
  Mode mode = Mode::kFixed;
  int order = 7;
  double tol = 1e-12;
  static TruncationPolicy fixed(int order);
  static TruncationPolicy adaptive(double tol = 1e-12);
};

struct OrderEstimate {
  int order = 0;
  bool converged = true;
};

double bessel_i0(double x);

// Smallest N in [8, 64] whose unit-boundary tail at max_abs_rho is below tol
// ({64, false} when none).  `length` is unused, as in the reference.
OrderEstimate estimate_order(double max_abs_rho, std::size_t length, double tol);

struct ErrorBoundInputs {
  std::size_t family_size = 1;
  std::size_t length = 2;
  double max_abs_increment_product = 0;
  int order = 7;
};

double gram_error_bound(const ErrorBoundInputs& inputs);

}  // namespace sigker
