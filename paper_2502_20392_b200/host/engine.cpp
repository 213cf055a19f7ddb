// The engine entry points of the drop-in C++ API (reference
// wavefront.cpp:196-237, gram.cpp:16-117) on top of the B200 C-ABI.
// Status codes come back as the reference's exception types.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>

#include "sigker/errors.hpp"
#include "sigker/gram.hpp"
#include "sigker/wavefront.hpp"
#include "sigker_b200.h"

namespace sigker {
namespace {

[[noreturn]] void rethrow(const sk_status& st) {
  switch (st.code) {
    case SK_INVALID_ARGUMENT:
      throw std::invalid_argument(st.message);
    case SK_NUMERIC_OVERFLOW:
      throw NumericOverflowError(st.message, st.tile_k, st.tile_l);
    case SK_INCONSISTENT_BOUNDARY:
      throw InconsistentBoundaryError(st.message);
    case SK_CUDA_ERROR:
      throw DeviceError(st.message);
    default:
      throw std::runtime_error(st.message);
  }
}

void check(int rc, sk_status& st) {
  if (rc != SK_OK) {
    if (st.code == SK_OK) st.code = rc;
    rethrow(st);
  }
}

uint32_t flags_of(const PropagateOptions& o) {
  return (o.strict_corner ? SK_STRICT_CORNER : 0u) | (tile::detail::w_fault_for_testing() ? SK_W_FAULT : 0u);
}

// wavefront.cpp live-series counter, closed form (derivation in sk_capi.cu
// peak_live_closed_form)
std::size_t peak_live(std::size_t rows, std::size_t cols) {
  const std::size_t m = std::min(rows, cols), big = std::max(rows, cols);
  return 2 * m + (big > m ? 1 : 0);
}

KernelResult run(const TimeSeries& x, const TimeSeries& y, int order, const PropagateOptions& options, bool grid) {
  if (x.dim() != y.dim()) throw std::invalid_argument("propagate: series dimensions differ");
  KernelResult r;
  r.order = order;
  if (grid) r.grid.assign(x.length() * y.length(), 0.0);
  sk_status st{};
  uint64_t pk = 0;
  check(sk_propagate(x.values().data(), x.length(), y.values().data(), y.length(), x.dim(), order,
                     flags_of(options), &r.value, &pk, grid ? r.grid.data() : nullptr, nullptr, &st),
        st);
  r.tiles_processed = (x.length() - 1) * (y.length() - 1);
  r.peak_live_series = static_cast<std::size_t>(pk);
  if (grid) {
    r.grid_rows = x.length();
    r.grid_cols = y.length();
  }
  return r;
}

}  // namespace

KernelResult propagate(const TimeSeries& x, const TimeSeries& y, int order, const PropagateOptions& options) {
  return run(x, y, order, options, false);
}

KernelResult propagate_grid(const TimeSeries& x, const TimeSeries& y, int order, const PropagateOptions& options) {
  return run(x, y, order, options, true);
}

KernelResult propagate_with_policy(const TimeSeries& x, const TimeSeries& y, const TruncationPolicy& policy,
                                   const PropagateOptions& options) {
  if (policy.mode == TruncationPolicy::Mode::kFixed) return propagate(x, y, policy.order, options);
  const PairwiseResult pr = pairwise({x}, {y}, policy, options);
  if (!pr.failures.empty())
    throw NumericOverflowError(pr.failures[0].message, pr.failures[0].tile_k, pr.failures[0].tile_l);
  KernelResult r;
  r.value = pr.values[0];
  r.order = pr.orders[0];
  r.order_converged = pr.converged[0];
  r.tiles_processed = (x.length() - 1) * (y.length() - 1);
  r.peak_live_series = peak_live(y.length() - 1, x.length() - 1);
  return r;
}

std::pair<tile::BoundarySeries, tile::BoundarySeries> step_tile(double delta, const tile::BoundarySeries& alpha,
                                                                const tile::BoundarySeries& beta, int order) {
  if (order < 0 || order > tile::kMaxOrder) throw std::invalid_argument("step_tile: order must lie in [0, 64]");
  const std::size_t n = static_cast<std::size_t>(order) + 1;
  if (alpha.a.size() < n || beta.a.size() < n)
    throw std::invalid_argument("step_tile: boundary series shorter than the order");
  tile::BoundarySeries up{tile::BoundaryAxis::AlongU, std::vector<double>(n)};
  tile::BoundarySeries right{tile::BoundaryAxis::AlongV, std::vector<double>(n)};
  sk_status st{};
  check(sk_step_tile(delta, alpha.a.data(), beta.a.data(), order, up.a.data(), right.a.data(), nullptr, &st), st);
  return {std::move(up), std::move(right)};
}

PairwiseResult pairwise(const std::vector<TimeSeries>& xs, const std::vector<TimeSeries>& ys,
                        const TruncationPolicy& policy, const PropagateOptions& options) {
  if (xs.size() != ys.size()) throw std::invalid_argument("pairwise: xs and ys differ in count");
  PairwiseResult out;
  const std::size_t np = xs.size();
  if (np == 0) return out;
  const std::size_t lx = xs[0].length(), ly = ys[0].length(), d = xs[0].dim();
  std::vector<double> bx, by;
  bx.reserve(np * lx * d);
  by.reserve(np * ly * d);
  for (std::size_t k = 0; k < np; ++k) {
    if (xs[k].length() != lx || ys[k].length() != ly || xs[k].dim() != d || ys[k].dim() != d)
      throw std::invalid_argument("pairwise: all xs (ys) must share one shape");
    bx.insert(bx.end(), xs[k].values().begin(), xs[k].values().end());
    by.insert(by.end(), ys[k].values().begin(), ys[k].values().end());
  }
  out.values.assign(np, 0.0);
  out.orders.assign(np, 0);
  std::vector<int> conv(np, 1);
  std::vector<sk_status> per(np);
  sk_status st{};
  const bool adaptive = policy.mode == TruncationPolicy::Mode::kAdaptive;
  check(sk_pairwise(bx.data(), lx, by.data(), ly, np, d, adaptive ? 1 : 0, policy.order, policy.tol,
                    flags_of(options), out.values.data(), out.orders.data(), conv.data(), nullptr, per.data(), &st),
        st);
  out.converged.assign(conv.begin(), conv.end());
  for (std::size_t k = 0; k < np; ++k) {
    if (per[k].code == SK_INCONSISTENT_BOUNDARY) rethrow(per[k]);
    if (per[k].code != SK_OK) out.failures.push_back({k, per[k].tile_k, per[k].tile_l, per[k].message});
  }
  return out;
}

GramResult gram_matrix(const std::vector<TimeSeries>& family, const GramOptions& options) {
  if (family.empty()) throw std::invalid_argument("gram_matrix: family must be nonempty");
  const std::size_t dim = family.front().dim();
  std::size_t max_len = 2;
  for (const auto& ts : family) {
    if (ts.dim() != dim) throw std::invalid_argument("gram_matrix: mixed dimensions in family");
    max_len = std::max(max_len, ts.length());
  }
  const std::size_t m = family.size();
  std::vector<double> buf;
  buf.reserve(m * max_len * dim);
  for (const auto& ts : family) {
    const TimeSeries p = pad_to_length(ts, max_len);
    buf.insert(buf.end(), p.values().begin(), p.values().end());
  }
  const bool adaptive = options.policy.mode == TruncationPolicy::Mode::kAdaptive;
  const bool scan = adaptive || options.compute_bound;
  GramResult r;
  r.size = m;
  r.adaptive = adaptive;
  r.values.assign(m * m, std::numeric_limits<double>::quiet_NaN());
  r.orders.assign(m * m, 0);
  int conv = 1;
  double maxp = 0.0;
  sk_status st{};
  const uint32_t flags = (options.strict_corner ? SK_STRICT_CORNER : 0u) |
                         (tile::detail::w_fault_for_testing() ? SK_W_FAULT : 0u);
  // the calling thread's failure records of its last sk_gram call (sparse)
  auto take_failures = [](std::size_t n, std::vector<GramEntryError>& out) {
    std::vector<sk_gram_failure> buf(n);
    n = sk_gram_failures(buf.data(), n);
    for (std::size_t k = 0; k < n; ++k) out.push_back({buf[k].row, buf[k].col, buf[k].status.message});
  };
  const auto t0 = std::chrono::steady_clock::now();
  const std::size_t nd = options.devices.size();
  if (nd <= 1) {
    if (nd == 1) check(sk_set_device(options.devices[0], &st), st);
    std::size_t nf = 0;
    check(sk_gram(buf.data(), m, max_len, dim, adaptive ? 1 : 0, options.policy.order, options.policy.tol, flags,
                  scan ? 1 : 0, options.shard, options.nshards, r.values.data(), r.orders.data(), nullptr, &maxp,
                  &conv, &nf, &st),
          st);
    take_failures(nf, r.failures);
  } else {
    // one host thread per device, each a sub-shard (shard * nd + k of nshards * nd);
    // every thread owns its context, so the calls run concurrently
    struct Part {
      std::vector<double> values;
      std::vector<int> orders;
      std::vector<GramEntryError> failures;
      double maxp = 0.0;
      int conv = 1;
      sk_status st{};
      int rc = SK_OK;
    };
    std::vector<Part> parts(nd);
    std::vector<std::thread> pool;
    for (std::size_t k = 0; k < nd; ++k)
      pool.emplace_back([&, k] {
        Part& pt = parts[k];
        pt.values.assign(m * m, 0.0);
        pt.orders.assign(m * m, 0);
        pt.rc = sk_set_device(options.devices[k], &pt.st);
        std::size_t nf = 0;
        if (pt.rc == SK_OK)
          pt.rc = sk_gram(buf.data(), m, max_len, dim, adaptive ? 1 : 0, options.policy.order, options.policy.tol,
                          flags, scan ? 1 : 0, options.shard * nd + k, options.nshards * nd, pt.values.data(),
                          pt.orders.data(), nullptr, &pt.maxp, &pt.conv, &nf, &pt.st);
        if (pt.rc == SK_OK) take_failures(nf, pt.failures);
      });
    for (auto& t : pool) t.join();
    for (Part& pt : parts) check(pt.rc, pt.st);
    // entry t of the upper triangle (row-major) belongs to the sub-shard whose range holds it
    std::size_t t = 0;
    std::vector<std::pair<std::size_t, std::size_t>> ranges(nd);
    for (std::size_t k = 0; k < nd; ++k)
      sk_gram_shard_range(m, options.shard * nd + k, options.nshards * nd, &ranges[k].first, &ranges[k].second);
    for (std::size_t i = 0; i < m; ++i)
      for (std::size_t j = i; j < m; ++j, ++t)
        for (std::size_t k = 0; k < nd; ++k)
          if (t >= ranges[k].first && t < ranges[k].second) {
            for (const std::size_t e : {i * m + j, j * m + i}) {
              r.values[e] = parts[k].values[e];
              r.orders[e] = parts[k].orders[e];
            }
            break;
          }
    // sub-shards are consecutive row-major ranges: concatenation keeps the order
    for (const Part& pt : parts) {
      maxp = std::max(maxp, pt.maxp);
      conv = conv && pt.conv;
      r.failures.insert(r.failures.end(), pt.failures.begin(), pt.failures.end());
    }
  }
  r.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  r.orders_converged = conv != 0;
  int lo = std::numeric_limits<int>::max(), hi = 0;
  std::size_t ok = 0;
  for (std::size_t e = 0; e < m * m; ++e) {
    if (r.orders[e] > 0) {
      lo = std::min(lo, r.orders[e]);
      hi = std::max(hi, r.orders[e]);
    }
    if (!std::isnan(r.values[e])) ++ok;
  }
  r.min_order = hi > 0 ? lo : 0;
  r.max_order = hi;
  r.peak_live_series = ok ? peak_live(max_len - 1, max_len - 1) : 0;
  if (scan) r.max_abs_increment_product = maxp;
  if (options.compute_bound) r.bound = gram_error_bound({m, max_len, r.max_abs_increment_product, r.min_order});
  return r;
}

MapeResult mape(std::span<const double> values, std::span<const double> reference) {
  if (values.size() != reference.size() || values.empty())
    throw std::invalid_argument("mape: shapes differ or empty input");
  MapeResult out;
  double sum = 0.0;
  std::size_t used = 0;
  for (std::size_t k = 0; k < values.size(); ++k) {
    if (reference[k] == 0.0) {
      ++out.excluded;
      continue;
    }
    sum += std::abs(values[k] - reference[k]) / std::abs(reference[k]);
    ++used;
  }
  if (used == 0) throw std::invalid_argument("mape: every reference entry is zero");
  out.value = sum / static_cast<double>(used);
  return out;
}

}  // namespace sigker
