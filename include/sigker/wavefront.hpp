// sigker/wavefront.hpp -- the signature-kernel engine of the drop-in C++ API
// (reference wavefront.hpp:13-60), executed by the B200 banded sweep through
// the C-ABI (sigker_b200.h).
#pragma once

#include <cstddef>
#include <string>
#include <utility>
#include <vector>

#include "sigker/tile_series.hpp"
#include "sigker/time_series.hpp"
#include "sigker/truncation.hpp"

namespace sigker {

struct PropagateOptions {
  unsigned threads = 1;            // advisory on the GPU (results never depend on it)
  bool reverse_diagonals = false;  // advisory on the GPU (results never depend on it)
  bool strict_corner = true;       // the reference's InconsistentBoundaryError check
};

struct KernelResult {
  double value = 1.0;
  int order = 0;
  bool order_converged = true;
  std::size_t tiles_processed = 0;
  std::size_t peak_live_series = 0;
  std::size_t grid_rows = 0;
  std::size_t grid_cols = 0;
  std::vector<double> grid;
};

KernelResult propagate(const TimeSeries& x, const TimeSeries& y, int order, const PropagateOptions& options = {});
KernelResult propagate_grid(const TimeSeries& x, const TimeSeries& y, int order,
                            const PropagateOptions& options = {});
KernelResult propagate_with_policy(const TimeSeries& x, const TimeSeries& y, const TruncationPolicy& policy,
                                   const PropagateOptions& options = {});
std::pair<tile::BoundarySeries, tile::BoundarySeries> step_tile(double delta, const tile::BoundarySeries& alpha,
                                                                const tile::BoundarySeries& beta, int order);

// Additions: batched independent pairs, each exactly
// propagate_with_policy(xs[k], ys[k]); overflowing pairs are NaN and listed.
struct PairFailure {
  std::size_t index = 0;
  std::size_t tile_k = 0, tile_l = 0;
  std::string message;
};
struct PairwiseResult {
  std::vector<double> values;
  std::vector<int> orders;
  std::vector<bool> converged;
  std::vector<PairFailure> failures;
};
PairwiseResult pairwise(const std::vector<TimeSeries>& xs, const std::vector<TimeSeries>& ys,
                        const TruncationPolicy& policy, const PropagateOptions& options = {});

}  // namespace sigker
