/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the tilewise power-series
 * signature-kernel path.  A plain-C restatement of the reference engine
 * (/root/reference/proj, "sigker"), used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER.  Nothing on the product
 * path (paper_2502_20392_b200/) links or calls this file.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libsigker_ref.so, built from the reference
 * sources by oracle/Makefile) and against the committed golden fixtures in
 * tests/golden/ (generated from the reference by oracle/make_golden.py).
 *
 * Compiled with -ffp-contract=off so every a*b+c rounds twice, exactly like
 * the reference's shipped flags (-O3 -DNDEBUG, no -march => no FMA).
 *
 * Each function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_ORDER 64 /* tile_series.hpp:12 kMaxOrder */

/* Status codes shared with include/sigker_b200.h */
enum { OR_OK = 0, OR_INVALID = 1, OR_OVERFLOW = 2, OR_INCONSISTENT = 3 };

typedef struct {
  int code;
  uint64_t tile_k, tile_l; /* 1-based, k along the first series */
  char message[256];
} or_status;

static void st_set(or_status* st, int code, uint64_t k, uint64_t l, const char* msg) {
  if (!st) return;
  st->code = code;
  st->tile_k = k;
  st->tile_l = l;
  strncpy(st->message, msg, sizeof st->message - 1);
  st->message[sizeof st->message - 1] = 0;
}

/* ---------------------------------------------------------------- datagen */
/* datagen.cpp:12-18 splitmix64 */
static uint64_t splitmix64(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

typedef struct {
  uint64_t s[4];
  double spare;
  int has_spare;
} or_rng;

/* datagen.cpp:42-45 */
void or_rng_init(or_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&sm);
  r->spare = 0.0;
  r->has_spare = 0;
}

or_rng* or_rng_new(uint64_t seed) {
  or_rng* r = (or_rng*)malloc(sizeof(or_rng));
  or_rng_init(r, seed);
  return r;
}
void or_rng_free(or_rng* r) { free(r); }

/* datagen.cpp:47-57 xoshiro256++ */
uint64_t or_rng_next_u64(or_rng* r) {
  const uint64_t result = rotl(r->s[0] + r->s[3], 23) + r->s[0];
  const uint64_t t = r->s[1] << 17;
  r->s[2] ^= r->s[0];
  r->s[3] ^= r->s[1];
  r->s[1] ^= r->s[2];
  r->s[0] ^= r->s[3];
  r->s[2] ^= t;
  r->s[3] = rotl(r->s[3], 45);
  return result;
}

/* datagen.cpp:59 */
double or_rng_uniform01(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* datagen.cpp:61-76 polar Box-Muller with a cached spare */
double or_rng_gaussian(or_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * or_rng_uniform01(r) - 1.0;
    v = 2.0 * or_rng_uniform01(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double f = sqrt(-2.0 * log(s) / s);
  r->spare = v * f;
  r->has_spare = 1;
  return u * f;
}

/* datagen.cpp:78-88 */
int or_brownian(size_t len, size_t dim, uint64_t seed, double* out) {
  if (len < 2 || dim < 1) return OR_INVALID;
  or_rng r;
  or_rng_init(&r, seed);
  const double sd = sqrt(1.0 / (double)(len - 1));
  memset(out, 0, len * dim * sizeof(double));
  for (size_t k = 1; k < len; ++k)
    for (size_t c = 0; c < dim; ++c) out[k * dim + c] = out[(k - 1) * dim + c] + sd * or_rng_gaussian(&r);
  return OR_OK;
}

/* datagen.cpp:23-38 */
static int cholesky(double* a, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = 0; j <= i; ++j) {
      double sum = a[i * n + j];
      for (size_t k = 0; k < j; ++k) sum -= a[i * n + k] * a[j * n + k];
      if (i == j) {
        if (sum <= 0.0) return 0;
        a[i * n + i] = sqrt(sum);
      } else {
        a[i * n + j] = sum / a[j * n + j];
      }
    }
    for (size_t j = i + 1; j < n; ++j) a[i * n + j] = 0.0;
  }
  return 1;
}

/* datagen.cpp:90-125 */
int or_fbm(size_t len, size_t dim, double hurst, uint64_t seed, double* out) {
  if (len < 2 || len > 4096 || dim < 1 || !(hurst > 0.0 && hurst < 1.0)) return OR_INVALID;
  const size_t n = len - 1;
  double* cov = (double*)malloc(n * n * sizeof(double));
  const double h2 = 2.0 * hurst;
  for (size_t i = 0; i < n; ++i) {
    const double ti = (double)(i + 1) / (double)(len - 1);
    for (size_t j = 0; j < n; ++j) {
      const double tj = (double)(j + 1) / (double)(len - 1);
      cov[i * n + j] = 0.5 * (pow(ti, h2) + pow(tj, h2) - pow(fabs(ti - tj), h2));
    }
  }
  if (!cholesky(cov, n)) {
    free(cov);
    return 4;
  }
  or_rng r;
  or_rng_init(&r, seed);
  memset(out, 0, len * dim * sizeof(double));
  double* z = (double*)malloc(n * sizeof(double));
  for (size_t c = 0; c < dim; ++c) {
    for (size_t k = 0; k < n; ++k) z[k] = or_rng_gaussian(&r);
    for (size_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (size_t k = 0; k <= i; ++k) acc += cov[i * n + k] * z[k];
      out[(i + 1) * dim + c] = acc;
    }
  }
  free(z);
  free(cov);
  return OR_OK;
}

/* tests/helpers.hpp:17-33 random_series (test fixture generator) */
void or_random_series(or_rng* r, size_t len, size_t dim, double max_increment_norm, double* out) {
  double* step = (double*)malloc(dim * sizeof(double));
  memset(out, 0, len * dim * sizeof(double));
  for (size_t k = 1; k < len; ++k) {
    double norm2 = 0.0;
    for (size_t c = 0; c < dim; ++c) {
      step[c] = or_rng_gaussian(r);
      norm2 += step[c] * step[c];
    }
    const double target = max_increment_norm * or_rng_uniform01(r);
    const double scale = norm2 > 0.0 ? target / sqrt(norm2) : 0.0;
    for (size_t c = 0; c < dim; ++c) out[k * dim + c] = out[(k - 1) * dim + c] + scale * step[c];
  }
  free(step);
}

/* ------------------------------------------------------------ increments */
/* time_series.cpp:32-42 */
static double* increments(const double* v, size_t len, size_t dim) {
  double* out = (double*)malloc((len - 1) * dim * sizeof(double) + 8);
  for (size_t k = 0; k + 1 < len; ++k)
    for (size_t i = 0; i < dim; ++i) out[k * dim + i] = v[(k + 1) * dim + i] - v[k * dim + i];
  return out;
}

/* time_series.cpp:54-62 (sequential in c, no FMA) */
static double rho(const double* a, const double* b, size_t dim) {
  double acc = 0.0;
  for (size_t i = 0; i < dim; ++i) acc += a[i] * b[i];
  return acc;
}

/* time_series.cpp:64-73 */
int or_max_abs_rho(const double* x, size_t lx, const double* y, size_t ly, size_t dim, double* out) {
  if (lx < 2 || ly < 2 || dim < 1) return OR_INVALID;
  double* xi = increments(x, lx, dim);
  double* yi = increments(y, ly, dim);
  double best = 0.0;
  for (size_t k = 0; k + 1 < lx; ++k)
    for (size_t l = 0; l + 1 < ly; ++l) {
      const double r = fabs(rho(xi + k * dim, yi + l * dim, dim));
      if (best < r) best = r; /* std::max(best, r) */
    }
  free(xi);
  free(yi);
  *out = best;
  return OR_OK;
}

/* ------------------------------------------------------------ tile algebra */
static double g_fact[171];
static int g_fact_ready = 0;

/* tile_series.cpp:19-27 */
static const double* factorials(void) {
  if (!g_fact_ready) {
    g_fact[0] = 1.0;
    for (int k = 1; k < 171; ++k) g_fact[k] = g_fact[k - 1] * (double)k;
    g_fact_ready = 1;
  }
  return g_fact;
}

/* tile_series.cpp:41-53 (without the fault hook) */
void or_build_W(int order, double* w) {
  const double* fact = factorials();
  const int n = order + 1;
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) {
      const double v = fact[j - i] / (fact[j] * fact[i]);
      w[i * n + j] = v;
      w[j * n + i] = v;
    }
}

/* tile_series.cpp:70-75; returns nonzero when the reference would throw */
int or_corner_mismatch(double a0, double b0) {
  double scale = 1.0;
  if (fabs(a0) > scale) scale = fabs(a0);
  if (fabs(b0) > scale) scale = fabs(b0);
  return fabs(a0 - b0) > 1e-9 * scale;
}

/* wavefront.cpp:35-59 fused_tile_step (corner check done by the caller);
 * returns the tile total. */
static double fused_tile_step(double delta, const double* alpha, const double* beta, const double* w,
                              int order, double* out_alpha, double* out_beta) {
  const int n = order + 1;
  double pw[OR_MAX_ORDER + 1];
  pw[0] = 1.0;
  for (int m = 1; m < n; ++m) pw[m] = pw[m - 1] * delta;
  for (int j = 0; j < n; ++j) out_beta[j] = 0.0;
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* wrow = w + (size_t)i * n;
    double row_sum = 0.0;
    for (int j = 0; j < n; ++j) {
      const double b = (i >= j) ? alpha[i - j] : beta[j - i];
      const double val = b * (pw[i < j ? i : j] * wrow[j]);
      row_sum += val;
      out_beta[j] += val;
    }
    out_alpha[i] = row_sum;
    total += row_sum;
  }
  return total;
}

/* wavefront.cpp:223-237 step_tile; returns total */
double or_step_tile(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                    double* out_beta) {
  double w[(OR_MAX_ORDER + 1) * (OR_MAX_ORDER + 1)];
  or_build_W(order, w);
  return fused_tile_step(delta, alpha, beta, w, order, out_alpha, out_beta);
}

/* wavefront.cpp:19-30, 107, 111-125, 175-176: the 1-thread sequence of the
 * live-series counter, simulated literally tile by tile. */
uint64_t or_peak_live(size_t rows, size_t cols) {
  long cur = 0, peak = 0;
#define OR_ADD(n_)                 \
  do {                             \
    cur += (n_);                   \
    if (cur > peak) peak = cur;    \
  } while (0)
  const size_t diagonals = rows + cols - 1;
  /* prefill(0) */
  OR_ADD(1);
  OR_ADD(1);
  for (size_t d = 0; d < diagonals; ++d) {
    const size_t start = d >= cols ? d - (cols - 1) : 0;
    const size_t end = d < rows - 1 ? d : rows - 1;
    if (d + 1 < diagonals) {
      if (d + 1 <= cols - 1) OR_ADD(1);
      if (d + 1 <= rows - 1) OR_ADD(1);
    }
    for (size_t i = start; i <= end; ++i) {
      const size_t j = d - i;
      cur -= 2;
      OR_ADD((i + 1 < rows ? 1 : 0) + (j + 1 < cols ? 1 : 0));
    }
  }
#undef OR_ADD
  return (uint64_t)peak;
}

/* wavefront.cpp:70-192 run(): anti-diagonal sweep, 1-thread tile order.
 * check_corner = 1 restates the reference exactly (throws
 * InconsistentBoundaryError via status 3); 0 is the check-free restatement
 * used where the reference throws.  The boundary
 * series are kept per column (alpha) and per row (beta) instead of the
 * reference's diagonal slots; tiles on one diagonal touch disjoint entries,
 * so the arithmetic and its order per tile are unchanged. */
/* Instrumentation of the same sweep (results are unchanged by it):
 *   knots/knot_vals: K at grid points (a, a) for each a in knots (the total of
 *     tile (a-1, a-1)); entries beyond the grid are left untouched;
 *   corner: worst |alpha0-beta0| / max(1,|alpha0|,|beta0|) over all tiles, and
 *     the first tile (diagonal order, 1-based k along x) where it exceeds 1e-9
 *     -- the tile at which the reference would throw (tile_series.cpp:70-75). */
typedef struct {
  const size_t* knots;
  size_t nknots;
  double* knot_vals;
  double max_corner_rel;
  uint64_t corner_k, corner_l;
} or_probe;

static int propagate_core(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                          int check_corner, double* value, uint64_t* peak_live, double* grid_or_null,
                          or_status* st, or_probe* pr);

int or_propagate(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                 int check_corner, double* value, uint64_t* peak_live, double* grid_or_null,
                 or_status* st) {
  return propagate_core(x, lx, y, ly, dim, order, check_corner, value, peak_live, grid_or_null, st, NULL);
}

int or_propagate_probe(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                       int check_corner, const size_t* knots, size_t nknots, double* knot_vals,
                       double* max_corner_rel, uint64_t* corner_k, uint64_t* corner_l, double* value,
                       or_status* st) {
  or_probe pr = {knots, nknots, knot_vals, 0.0, 0, 0};
  const int rc = propagate_core(x, lx, y, ly, dim, order, check_corner, value, NULL, NULL, st, &pr);
  *max_corner_rel = pr.max_corner_rel;
  *corner_k = pr.corner_k;
  *corner_l = pr.corner_l;
  return rc;
}

static int propagate_core(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                          int check_corner, double* value, uint64_t* peak_live, double* grid_or_null,
                          or_status* st, or_probe* pr) {
  if (st) memset(st, 0, sizeof *st);
  if (lx < 2 || ly < 2) {
    st_set(st, OR_INVALID, 0, 0, "propagate: both series need length >= 2");
    return OR_INVALID;
  }
  if (order < 1 || order > OR_MAX_ORDER) {
    st_set(st, OR_INVALID, 0, 0, "propagate: order must lie in [1, 64]");
    return OR_INVALID;
  }
  const size_t cols = lx - 1, rows = ly - 1;
  const int n = order + 1;
  double* xi = increments(x, lx, dim);
  double* yi = increments(y, ly, dim);
  double* w = (double*)malloc((size_t)n * n * sizeof(double));
  or_build_W(order, w);
  double* alpha = (double*)calloc(cols * n, sizeof(double)); /* bottom edge per column */
  double* beta = (double*)calloc(rows * n, sizeof(double));  /* left edge per row */
  for (size_t j = 0; j < cols; ++j) alpha[j * n] = 1.0;
  for (size_t i = 0; i < rows; ++i) beta[i * n] = 1.0;
  if (grid_or_null) {
    memset(grid_or_null, 0, lx * ly * sizeof(double));
    for (size_t a = 0; a < lx; ++a) grid_or_null[a * ly] = 1.0;
    for (size_t b = 0; b < ly; ++b) grid_or_null[b] = 1.0;
  }
  double out_a[OR_MAX_ORDER + 1], out_b[OR_MAX_ORDER + 1];
  double final_value = 1.0;
  int rc = OR_OK;
  const size_t diagonals = rows + cols - 1;
  for (size_t d = 0; d < diagonals && rc == OR_OK; ++d) {
    const size_t start = d >= cols ? d - (cols - 1) : 0;
    const size_t end = d < rows - 1 ? d : rows - 1;
    for (size_t i = start; i <= end; ++i) {
      const size_t j = d - i;
      const double delta = rho(xi + j * dim, yi + i * dim, dim);
      if (!(fabs(delta) <= 1.25e5)) { /* wavefront.cpp:17,150-155 */
        st_set(st, OR_OVERFLOW, j + 1, i + 1,
               "increment product exceeds double range at any order; rescale the inputs");
        rc = OR_OVERFLOW;
        break;
      }
      double* a = alpha + j * n;
      double* b = beta + i * n;
      if (pr) {
        double sc = 1.0;
        if (fabs(a[0]) > sc) sc = fabs(a[0]);
        if (fabs(b[0]) > sc) sc = fabs(b[0]);
        const double rel = fabs(a[0] - b[0]) / sc;
        if (rel > pr->max_corner_rel) pr->max_corner_rel = rel;
        if (pr->corner_k == 0 && or_corner_mismatch(a[0], b[0])) {
          pr->corner_k = j + 1;
          pr->corner_l = i + 1;
        }
      }
      if (check_corner && or_corner_mismatch(a[0], b[0])) { /* tile_series.cpp:70-75 */
        st_set(st, OR_INCONSISTENT, j + 1, i + 1, "boundary series disagree at the shared corner");
        rc = OR_INCONSISTENT;
        break;
      }
      const double total = fused_tile_step(delta, a, b, w, order, out_a, out_b);
      if (!isfinite(total)) { /* wavefront.cpp:169-173 */
        st_set(st, OR_OVERFLOW, j + 1, i + 1, "non-finite series; rescale the inputs or reduce the order");
        rc = OR_OVERFLOW;
        break;
      }
      memcpy(a, out_a, n * sizeof(double));
      memcpy(b, out_b, n * sizeof(double));
      if (grid_or_null) grid_or_null[(j + 1) * ly + (i + 1)] = total;
      if (i + 1 == rows && j + 1 == cols) final_value = total;
      if (pr && i == j)
        for (size_t q = 0; q < pr->nknots; ++q)
          if (pr->knots[q] == i + 1) pr->knot_vals[q] = total;
    }
  }
  if (rc == OR_OK) {
    *value = final_value;
    if (peak_live) *peak_live = or_peak_live(rows, cols);
  }
  free(xi);
  free(yi);
  free(w);
  free(alpha);
  free(beta);
  return rc;
}

/* --------------------------------------------------------------- truncation */
/* truncation.cpp:41-55 with tile_coeffs (tile_series.cpp:123-132) at unit
 * boundaries: entry c[i][j] = B[i][j] * (A[i][j] * W[i][j]). */
int or_estimate_order(double max_abs_rho, double tol, int* order, int* converged) {
  if (!(tol > 0.0)) return OR_INVALID;
  if (max_abs_rho < 0.0 || !isfinite(max_abs_rho)) return OR_INVALID;
  const double* fact = factorials();
  for (int n = 8; n <= OR_MAX_ORDER; ++n) {
    const int sz = n + 1;
    /* A = delta^min(i,j) by cumulative powers (tile_series.cpp:55-68) */
    double pw[OR_MAX_ORDER + 1];
    pw[0] = 1.0;
    for (int m = 1; m < sz; ++m) pw[m] = pw[m - 1] * max_abs_rho;
    double tail = 0.0;
    for (int j = 0; j <= n; ++j) {
      const double b = (n == j) ? 1.0 : 0.0; /* unit alpha: alpha[n-j] */
      const int mn = n < j ? n : j;
      const int hi = n > j ? n : j, lo = n < j ? n : j;
      const double wv = fact[hi - lo] / (fact[hi] * fact[lo]);
      tail += b * (pw[mn] * wv);
    }
    for (int i = 0; i <= n; ++i) {
      const double b = (i == n) ? 1.0 : 0.0; /* i < n: unit beta[n-i] = 0 */
      const int mn = i < n ? i : n;
      const int hi = n > i ? n : i, lo = n < i ? n : i;
      const double wv = fact[hi - lo] / (fact[hi] * fact[lo]);
      tail += b * (pw[mn] * wv);
    }
    if (tail < tol) {
      *order = n;
      *converged = 1;
      return OR_OK;
    }
  }
  *order = OR_MAX_ORDER;
  *converged = 0;
  return OR_OK;
}

/* truncation.cpp:28-39 */
double or_bessel_i0(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 1000; ++k) {
    term *= q / ((double)k * (double)k);
    sum += term;
    if (term < sum * 2.220446049250313e-16) break;
  }
  return sum;
}

/* truncation.cpp:57-87 */
double or_gram_error_bound(size_t m, size_t len, double max_prod, int order) {
  const double lm1 = (double)(len - 1);
  const int n = order;
  const double max_x = lm1 * lm1 * max_prod;
  double gamma = 0.5 * (double)m;
  const size_t terms = 2 * len - 2;
  for (size_t nu = 0; nu <= terms; ++nu) gamma *= or_bessel_i0(2.0 * sqrt((double)nu * max_x) / lm1);
  const double zeta = (1.0 + (2.0 * lm1) / (n + 2.0)) * pow(2.0 / lm1, n + 1);
  const double* fact = factorials();
  if ((size_t)n + 1 < 171) {
    const double fac = fact[n + 1];
    return gamma * pow(max_x, n + 1) * zeta / (fac * fac);
  }
  const double log_tail = (n + 1) * log(max_x) - 2.0 * lgamma(n + 2.0);
  return gamma * zeta * exp(log_tail);
}

/* -------------------------------------------------------------------- gram */
/* gram.cpp:16-98, sequential pair order (results are thread-count independent,
 * test_gram.cpp:70-79).  family: m series of common length len.  Entries that
 * overflow stay NaN and are counted in *n_failures. */
int or_gram(const double* family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
            int check_corner, double* values, int* orders, double* max_prod, uint64_t* n_failures) {
  size_t fails = 0;
  double best = 0.0;
  for (size_t k = 0; k < m * m; ++k) {
    values[k] = NAN;
    orders[k] = 0;
  }
  for (size_t i = 0; i < m; ++i)
    for (size_t j = i; j < m; ++j) {
      const double* xi = family + i * len * dim;
      const double* xj = family + j * len * dim;
      int ord = order, conv = 1;
      if (adaptive) {
        double mr;
        or_max_abs_rho(xi, len, xj, len, dim, &mr);
        if (mr > best) best = mr;
        or_estimate_order(mr, tol, &ord, &conv);
      }
      double v;
      or_status st;
      const int rc = or_propagate(xi, len, xj, len, dim, ord, check_corner, &v, NULL, NULL, &st);
      if (rc == OR_OK) {
        values[i * m + j] = v;
        values[j * m + i] = v;
      } else if (rc == OR_OVERFLOW) {
        ++fails;
      } else {
        return rc;
      }
      orders[i * m + j] = ord;
      orders[j * m + i] = ord;
    }
  if (max_prod) *max_prod = best;
  if (n_failures) *n_failures = fails;
  return OR_OK;
}
