// Synthetic series generators -- the reference's datagen.hpp API (generators
// datagen.cpp:78-150, PRNG datagen.cpp:44-76), implemented in
// paper_2502_20392_b200/host/datagen.cpp.  Streams are bit-identical to the
// reference's for equal seeds (pinned by tests/golden/datagen.json).
#pragma once

#include <cstddef>
#include <cstdint>

#include "sigker/time_series.hpp"

namespace sigker::datagen {

// xoshiro256++ seeded by four splitmix64 outputs; uniform01 = top 53 bits
// * 2^-53; gaussian = polar Marsaglia method with the second variate cached.
class Rng {
 public:
  explicit Rng(std::uint64_t seed);
  std::uint64_t next_u64();
  double uniform01();
  double gaussian();

 private:
  std::uint64_t s_[4];
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// Brownian path from the origin, step variance 1/(length-1), coordinates of
// one step drawn consecutively.
TimeSeries brownian(std::size_t length, std::size_t dim, std::uint64_t seed);

// Exact fractional Brownian motion on the uniform grid (dense Cholesky of the
// covariance, length <= 4096), coordinate-major draws; NumericError when the
// factorization breaks down.
TimeSeries fbm(std::size_t length, std::size_t dim, double hurst, std::uint64_t seed);

// amplitude * sin(2 pi t / period + phase_c) + noise * N(0,1), t = k/(length-1);
// phases first (uniform on [0, 2 pi)), then the noise draws.
TimeSeries near_periodic(std::size_t length, std::size_t dim, double period, double amplitude, double noise,
                         std::uint64_t seed);

}  // namespace sigker::datagen

// C binding of brownian() (row-major length x dim into `out`; 0 on success).
extern "C" int sigker_datagen_brownian(std::size_t length, std::size_t dim, std::uint64_t seed, double* out);
