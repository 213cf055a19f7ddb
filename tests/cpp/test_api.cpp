// C++ drop-in API tests: the engine behaviours the reference pins in its unit
// suites (test_wavefront.cpp, test_gram.cpp, test_truncation.cpp), exercised
// through include/sigker/*.hpp on the B200 engine.  Run by
// tests/test_cpp_api.py (needs a GPU); prints one line per check group and
// exits non-zero on any failure.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "sigker/errors.hpp"
#include "sigker/gram.hpp"
#include "sigker/tile_series.hpp"
#include "sigker/time_series.hpp"
#include "sigker/truncation.hpp"
#include "sigker/wavefront.hpp"

using namespace sigker;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                       \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static bool close(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

// splitmix64-seeded xorshift for test inputs (independent of any library RNG)
struct TestRng {
  uint64_t s;
  explicit TestRng(uint64_t seed) : s(seed * 0x9E3779B97F4A7C15ULL + 1) {}
  double uniform() {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return static_cast<double>(s >> 11) * 0x1.0p-53;
  }
  TimeSeries series(std::size_t len, std::size_t dim, double cap) {
    std::vector<double> v(len * dim, 0.0);
    for (std::size_t k = 1; k < len; ++k)
      for (std::size_t c = 0; c < dim; ++c) v[k * dim + c] = v[(k - 1) * dim + c] + cap * (2.0 * uniform() - 1.0);
    return TimeSeries(std::move(v), dim);
  }
};

static TimeSeries s1(std::initializer_list<double> pts) { return TimeSeries(std::vector<double>(pts), 1); }

static double diag_series(double rho, int order) {
  double s = 0.0, f = 1.0;
  for (int i = 0; i <= order; ++i) {
    if (i > 0) f *= i;
    s += std::pow(rho, i) / (f * f);
  }
  return s;
}

int main() {
  std::printf("constant series / single tile\n");
  for (std::size_t len : {2u, 3u, 9u}) {
    const auto x = pad_to_length(TimeSeries({0.4, -1.0}, 2), len);
    const auto r = propagate(x, x, 12);
    CHECK(r.value == 1.0);
    CHECK(r.tiles_processed == (len - 1) * (len - 1));
  }
  const auto unit = s1({0.0, 1.0});
  for (double rho : {-4.0, -1.0, 0.5, 1.0, 4.0}) CHECK(close(propagate(unit, s1({0.0, rho}), 24).value,
                                                             diag_series(rho, 24), 1e-14));
  CHECK(close(propagate(unit, unit, 24).value, 2.2795853023360673, 1e-14));

  std::printf("collinear refinement, symmetry, positivity, monotone order\n");
  CHECK(close(propagate(s1({0.0, 0.5, 1.0}), s1({0.0, 0.5, 1.0}), 20).value, propagate(unit, unit, 20).value, 1e-12));
  TestRng rng(123);
  for (int t = 0; t < 8; ++t) {
    const auto x = rng.series(3 + t, 2, 0.8), y = rng.series(3 + t, 2, 0.8);
    const double xy = propagate(x, y, 24).value, yx = propagate(y, x, 24).value;
    CHECK(std::abs(xy - yx) <= 1e-12 * std::max(1.0, std::abs(xy)));
    CHECK(propagate(x, x, 24).value >= 1.0 - 1e-10);
  }
  const TimeSeries mono({0.0, 0.0, 0.7, 0.4, 1.1, 0.9, 2.0, 1.5}, 2);
  double prev = 0.0;
  for (int n : {4, 6, 8, 10, 12, 16}) {
    const double v = propagate(mono, mono, n).value;
    CHECK(v >= prev);
    prev = v;
  }

  std::printf("step_tile composes the tile algebra\n");
  TestRng r2(31);
  for (int t = 0; t < 25; ++t) {
    const int order = 2 + t % 14;
    tile::BoundarySeries a{tile::BoundaryAxis::AlongU, std::vector<double>(order + 1)};
    tile::BoundarySeries b{tile::BoundaryAxis::AlongV, std::vector<double>(order + 1)};
    a.a[0] = b.a[0] = 2.0 * r2.uniform() - 1.0;
    for (int k = 1; k <= order; ++k) {
      a.a[k] = (2.0 * r2.uniform() - 1.0) / (k * k + 1.0);
      b.a[k] = (2.0 * r2.uniform() - 1.0) / (k * k + 1.0);
    }
    const double delta = 6.0 * r2.uniform() - 3.0;
    const auto [up, right] = step_tile(delta, a, b, order);
    const auto c = tile::tile_coeffs(delta, a, b, order);
    CHECK(up.a == tile::top_boundary(c).a);
    CHECK(right.a == tile::right_boundary(c).a);
  }

  std::printf("grid output, rectangular inputs\n");
  const auto g = propagate_grid(unit, unit, 16);
  CHECK(g.grid.size() == 4 && g.grid[0] == 1.0 && g.grid[1] == 1.0 && g.grid[2] == 1.0 && g.grid[3] == g.value);
  const auto z = rng.series(7, 2, 1.0);
  const auto self = propagate_grid(z, z, 20);
  for (std::size_t a = 0; a < 7; ++a)
    for (std::size_t b = 0; b < 7; ++b) CHECK(close(self.grid[a * 7 + b], self.grid[b * 7 + a], 1e-12));
  const double rect = propagate(unit, s1({0.0, 0.3, 0.9}), 24).value;
  CHECK(close(rect, propagate(pad_to_length(unit, 3), s1({0.0, 0.3, 0.9}), 24).value, 1e-13));
  CHECK(close(rect, diag_series(0.9, 24), 1e-12));

  std::printf("argument validation and the overflow guard\n");
  CHECK(throws<std::invalid_argument>([&] { propagate(unit, TimeSeries({0.0, 0.0, 1.0, 1.0}, 2), 8); }));
  CHECK(throws<std::invalid_argument>([&] { propagate(unit, unit, 0); }));
  CHECK(throws<std::invalid_argument>([&] { propagate(unit, unit, 65); }));
  CHECK(throws<std::invalid_argument>([&] { propagate(TimeSeries({1.0}, 1), unit, 8); }));
  try {
    propagate(s1({0.0, 400.0}), s1({0.0, 400.0}), 24);
    CHECK(false);
  } catch (const NumericOverflowError& e) {
    CHECK(e.tile_k() == 1 && e.tile_l() == 1);
    CHECK(std::string(e.what()).find("rescale") != std::string::npos);
  }

  std::printf("truncation policy\n");
  const auto fixed = propagate_with_policy(unit, unit, TruncationPolicy::fixed(24));
  const auto adaptive = propagate_with_policy(unit, unit, TruncationPolicy::adaptive(1e-12));
  CHECK(fixed.order == 24 && adaptive.order == 10 && adaptive.order_converged);
  CHECK(std::abs(adaptive.value - fixed.value) < 1e-10);
  CHECK(estimate_order(0.0, 16, 1e-12).order == 8);
  CHECK(estimate_order(1.0, 16, 1e-12).order == 10);
  CHECK(!estimate_order(1e6, 16, 1e-12).converged && estimate_order(1e6, 16, 1e-12).order == 64);
  CHECK(throws<std::invalid_argument>([] { TruncationPolicy::fixed(0); }));
  CHECK(throws<std::invalid_argument>([] { TruncationPolicy::adaptive(0.0); }));
  CHECK(close(bessel_i0(2.0), 2.2795853023360673, 1e-15));

  std::printf("gram matrix\n");
  const auto constant = pad_to_length(s1({3.0, 3.0}), 4);
  CHECK(gram_matrix({constant}).values[0] == 1.0);
  const auto x6 = rng.series(6, 2, 1.0);
  const auto dup = gram_matrix({x6, x6}, {TruncationPolicy::fixed(16)});
  CHECK(dup.values[0] == dup.values[1] && dup.values[1] == dup.values[2] && dup.values[2] == dup.values[3]);
  CHECK(throws<std::invalid_argument>([] { gram_matrix({}); }));
  CHECK(throws<std::invalid_argument>([&] { gram_matrix({x6, s1({0.0, 1.0})}); }));
  std::vector<TimeSeries> fam;
  for (int k = 0; k < 5; ++k) fam.push_back(rng.series(9, 2, 0.7));
  const auto gm = gram_matrix(fam, {TruncationPolicy::fixed(20)});
  for (std::size_t i = 0; i < 5; ++i) {
    CHECK(gm.values[i * 5 + i] >= 1.0 - 1e-10);
    for (std::size_t j = 0; j < 5; ++j) CHECK(close(gm.values[i * 5 + j], gm.values[j * 5 + i], 1e-12));
  }
  for (std::size_t i = 0; i < 5; ++i)
    for (std::size_t j = i; j < 5; ++j) CHECK(close(gm.values[i * 5 + j], propagate(fam[i], fam[j], 20).value, 1e-10));
  {
    // GramOptions::devices: one host thread per listed GPU (here GPU 0 twice), merged bit for bit
    GramOptions two{TruncationPolicy::fixed(20)};
    two.devices = {0, 0};
    const auto g2 = gram_matrix(fam, two);
    CHECK(g2.values == gm.values && g2.orders == gm.orders);
  }
  const auto fail = gram_matrix({s1({0.0, 1.0}), s1({0.0, 1e4})}, {TruncationPolicy::fixed(8)});
  CHECK(!fail.failures.empty() && fail.failures.front().row == 1 && fail.failures.front().col == 1);
  CHECK(std::isnan(fail.values[3]) && std::isfinite(fail.values[0]) && std::isfinite(fail.values[1]));
  GramOptions bopt;
  bopt.policy = TruncationPolicy::fixed(12);
  bopt.compute_bound = true;
  const auto gb = gram_matrix(fam, bopt);
  CHECK(gb.max_abs_increment_product > 0.0 && !std::isnan(gb.bound));
  const std::vector<double> ref{2.0, -4.0, 8.0};
  CHECK(mape(ref, ref).value == 0.0);

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
