// TEST INFRASTRUCTURE ONLY (oracle). A C-ABI shim over the UNMODIFIED reference
// engine `sigker` (/root/reference/proj/src/*.cpp), compiled together with those
// sources by oracle/Makefile into oracle/_ref/libsigker_ref.so. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it. Nothing here is on the product path.
//
// Status codes (shared with the product C-ABI, include/sigker_b200.h):
//   0 ok, 1 std::invalid_argument, 2 NumericOverflowError,
//   3 InconsistentBoundaryError, 4 any other exception.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "sigker/datagen.hpp"
#include "sigker/errors.hpp"
#include "sigker/gram.hpp"
#include "sigker/thread_pool.hpp"
#include "sigker/tile_series.hpp"
#include "sigker/time_series.hpp"
#include "sigker/truncation.hpp"
#include "sigker/wavefront.hpp"

using namespace sigker;

namespace {

struct RefStatus {
  int code;
  uint64_t tile_k, tile_l;
  char message[256];
};

void set_msg(RefStatus* st, const char* m) {
  if (!st) return;
  std::strncpy(st->message, m, sizeof st->message - 1);
  st->message[sizeof st->message - 1] = 0;
}

template <class F>
int guarded(RefStatus* st, F&& f) {
  if (st) std::memset(st, 0, sizeof *st);
  try {
    f();
    return 0;
  } catch (const NumericOverflowError& e) {
    if (st) {
      st->code = 2;
      st->tile_k = e.tile_k();
      st->tile_l = e.tile_l();
      set_msg(st, e.what());
    }
    return 2;
  } catch (const InconsistentBoundaryError& e) {
    if (st) st->code = 3;
    set_msg(st, e.what());
    return 3;
  } catch (const std::invalid_argument& e) {
    if (st) st->code = 1;
    set_msg(st, e.what());
    return 1;
  } catch (const std::exception& e) {
    if (st) st->code = 4;
    set_msg(st, e.what());
    return 4;
  }
}

TimeSeries ts(const double* v, size_t len, size_t dim) {
  return TimeSeries(std::vector<double>(v, v + len * dim), dim);
}

}  // namespace

extern "C" {

int ref_propagate(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                  unsigned threads, int reverse, double* value, uint64_t* peak_live,
                  double* grid_or_null, RefStatus* st) {
  return guarded(st, [&] {
    PropagateOptions o;
    o.threads = threads;
    o.reverse_diagonals = reverse != 0;
    const auto tx = ts(x, lx, dim), ty = ts(y, ly, dim);
    const KernelResult r = grid_or_null ? propagate_grid(tx, ty, order, o) : propagate(tx, ty, order, o);
    *value = r.value;
    if (peak_live) *peak_live = r.peak_live_series;
    if (grid_or_null) std::memcpy(grid_or_null, r.grid.data(), r.grid.size() * sizeof(double));
  });
}

int ref_propagate_with_policy(const double* x, size_t lx, const double* y, size_t ly, size_t dim,
                              int adaptive, int order, double tol, unsigned threads, double* value,
                              int* order_out, int* converged, RefStatus* st) {
  return guarded(st, [&] {
    TruncationPolicy p = adaptive ? TruncationPolicy::adaptive(tol) : TruncationPolicy::fixed(order);
    PropagateOptions o;
    o.threads = threads;
    const KernelResult r = propagate_with_policy(ts(x, lx, dim), ts(y, ly, dim), p, o);
    *value = r.value;
    *order_out = r.order;
    *converged = r.order_converged ? 1 : 0;
  });
}

int ref_max_abs_rho(const double* x, size_t lx, const double* y, size_t ly, size_t dim, double* out,
                    RefStatus* st) {
  return guarded(st, [&] {
    const IncrementTable t(ts(x, lx, dim), ts(y, ly, dim));
    *out = t.max_abs_rho();
  });
}

int ref_estimate_order(double max_abs_rho, size_t length, double tol, int* order, int* converged,
                       RefStatus* st) {
  return guarded(st, [&] {
    const auto e = estimate_order(max_abs_rho, length, tol);
    *order = e.order;
    *converged = e.converged ? 1 : 0;
  });
}

int ref_step_tile(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                  double* out_beta, RefStatus* st) {
  return guarded(st, [&] {
    const size_t n = static_cast<size_t>(order) + 1;
    tile::BoundarySeries a{tile::BoundaryAxis::AlongU, std::vector<double>(alpha, alpha + n)};
    tile::BoundarySeries b{tile::BoundaryAxis::AlongV, std::vector<double>(beta, beta + n)};
    const auto [up, right] = step_tile(delta, a, b, order);
    std::memcpy(out_alpha, up.a.data(), n * sizeof(double));
    std::memcpy(out_beta, right.a.data(), n * sizeof(double));
  });
}

// family: m series of common length len (row-major len x dim each, contiguous).
int ref_gram(const double* family, size_t m, size_t len, size_t dim, int adaptive, int order,
             double tol, unsigned threads, int compute_bound, double* values, int* orders,
             double* max_abs_increment_product, double* bound, uint64_t* peak_live,
             int* orders_converged, uint64_t* n_failures, double* wall_seconds, RefStatus* st) {
  return guarded(st, [&] {
    std::vector<TimeSeries> fam;
    fam.reserve(m);
    for (size_t i = 0; i < m; ++i) fam.push_back(ts(family + i * len * dim, len, dim));
    GramOptions o;
    o.policy = adaptive ? TruncationPolicy::adaptive(tol) : TruncationPolicy::fixed(order);
    o.threads = threads;
    o.compute_bound = compute_bound != 0;
    const GramResult r = gram_matrix(fam, o);
    std::memcpy(values, r.values.data(), m * m * sizeof(double));
    std::memcpy(orders, r.orders.data(), m * m * sizeof(int));
    *max_abs_increment_product = r.max_abs_increment_product;
    *bound = r.bound;
    *peak_live = r.peak_live_series;
    *orders_converged = r.orders_converged ? 1 : 0;
    *n_failures = r.failures.size();
    *wall_seconds = r.wall_seconds;
  });
}

// Batched pairs the way gram.cpp:51-66 parallelises a family: a static
// ThreadPool split of the pair list, each pair a single-threaded
// propagate_with_policy. xs/ys: npairs series each of shape len x dim.
int ref_pairwise(const double* xs, const double* ys, size_t npairs, size_t len, size_t dim, int adaptive,
                 int order, double tol, unsigned threads, double* values, int* orders, RefStatus* st) {
  return guarded(st, [&] {
    ThreadPool pool(threads < 1 ? 1u : threads);
    const TruncationPolicy p = adaptive ? TruncationPolicy::adaptive(tol) : TruncationPolicy::fixed(order);
    pool.parallel_for(npairs, [&](unsigned, size_t lo, size_t hi) {
      for (size_t k = lo; k < hi; ++k) {
        const KernelResult r = propagate_with_policy(ts(xs + k * len * dim, len, dim),
                                                     ts(ys + k * len * dim, len, dim), p);
        values[k] = r.value;
        orders[k] = r.order;
      }
    });
  });
}

int ref_brownian(size_t len, size_t dim, uint64_t seed, double* out, RefStatus* st) {
  return guarded(st, [&] {
    const auto t = datagen::brownian(len, dim, seed);
    std::memcpy(out, t.values().data(), len * dim * sizeof(double));
  });
}

int ref_fbm(size_t len, size_t dim, double hurst, uint64_t seed, double* out, RefStatus* st) {
  return guarded(st, [&] {
    const auto t = datagen::fbm(len, dim, hurst, seed);
    std::memcpy(out, t.values().data(), len * dim * sizeof(double));
  });
}

int ref_gram_error_bound(size_t m, size_t len, double max_x, int order, double* out, RefStatus* st) {
  return guarded(st, [&] { *out = gram_error_bound({m, len, max_x, order}); });
}

double ref_bessel_i0(double x) { return bessel_i0(x); }

// Stream of gaussians / uniforms from datagen::Rng, for pinning the oracle's RNG.
int ref_rng_stream(uint64_t seed, size_t n, int gaussian, double* out) {
  datagen::Rng r(seed);
  for (size_t i = 0; i < n; ++i) out[i] = gaussian ? r.gaussian() : r.uniform01();
  return 0;
}

}  // extern "C"
