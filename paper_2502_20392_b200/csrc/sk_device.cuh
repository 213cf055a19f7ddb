// Device-side building blocks of the B200 tile solver.
//
// Tile map (reference: wavefront.cpp:35-59 fused_tile_step; spec form
// tile_series.cpp:123-171).  A tile with increment product delta, bottom-edge
// series alpha (a series in u) and left-edge series beta (a series in v) has
// coefficients
//     c[a][b] = B[a][b] * delta^min(a,b) * W[a][b],
//     B[a][b] = alpha[a-b] (a >= b) else beta[b-a],  W[a][b] = |a-b|!/(a! b!),
// and hands alpha'[a] = sum_b c[a][b] up, beta'[b] = sum_a c[a][b] right and
// total = sum c = K at the tile's far corner.
//
// The register kernels carry the series in FACTORIAL-SCALED form
// q[m] = m! alpha[m], r[m] = m! beta[m].  With p[m] = delta^m / m! and
// pw[m] = delta^m the map becomes (exact algebra; only the rounding order
// differs from the reference):
//     q'[a] = sum_{b=0..a} q[a-b] p[b]          + pw[a] * sum_{k=1..N-a} r[k] / (a+k)!
//     r'[b] = sum_{a=0..b-1} r[b-a] p[a]        + pw[b] * sum_{k=0..N-b} q[k] / (b+k)!
//     total = sum_a q'[a] / a!
// i.e. two triangular Toeplitz products (the convolutions with p) and two
// triangular Hankel products with constant 1/k! weights: ~2 (N+1)^2 DFMA per
// tile instead of the literal 3 (N+1)^2 FP64 instructions.  The diagonal entry
// a = b always takes alpha[0] (q[0]), never beta[0], as the reference's
// `i >= j` branch does.
#pragma once

#include <cstdint>

#include "sk_tables.cuh"

namespace skb {

constexpr int kMaxOrder = 64;        // tile_series.hpp:12
constexpr int kMaxRegOrder = 16;     // register-resident kernels cover N <= 16
constexpr double kDeltaOverflowLimit = 1.25e5;  // wavefront.cpp:17

// Error codes packed into the per-pair error key (lowest 2 bits).
constexpr unsigned kErrDelta = 1;     // |delta| > 1.25e5       (wavefront.cpp:150-155)
constexpr unsigned kErrCorner = 2;    // InconsistentBoundary   (tile_series.cpp:70-75)
constexpr unsigned kErrNonFinite = 3; // non-finite tile total  (wavefront.cpp:169-173)

// Key ordering = the reference's 1-thread throw order: diagonal d = i + j
// first, then row i within the diagonal (wavefront.cpp:133-144).
__device__ __forceinline__ unsigned long long err_key(unsigned i, unsigned j, unsigned code) {
  return (static_cast<unsigned long long>(i + j) << 32) | (static_cast<unsigned long long>(i) << 2) | code;
}

// tile_series.cpp:70-75
__device__ __forceinline__ bool corner_mismatch(double a0, double b0) {
  const double scale = fmax(1.0, fmax(fabs(a0), fabs(b0)));
  return fabs(a0 - b0) > 1e-9 * scale;
}

// Sequential non-FMA dot product in coordinate order: bit-identical to
// `acc += a[c] * b[c]` at the reference's shipped flags
// (wavefront.cpp:146-149, time_series.cpp:54-62).
template <int DP>
__device__ __forceinline__ double exact_dot(const double (&a)[DP], const double (&b)[DP]) {
  double acc = __dmul_rn(a[0], b[0]);
#pragma unroll
  for (int c = 1; c < DP; ++c) acc = __dadd_rn(acc, __dmul_rn(a[c], b[c]));
  return acc;
}

// Register tile step on scaled series (see header comment).  Returns total.
// `fault` flips the sign of the W[1][1] contribution (the reference's
// negative-control hook, tile_series.cpp:51-52).
template <int N>
__device__ __forceinline__ double tile_step_scaled(const double (&q)[N + 1], const double (&r)[N + 1],
                                                   double delta, double (&qo)[N + 1], double (&ro)[N + 1],
                                                   bool fault) {
  constexpr int n = N + 1;
  double pw[n], p[n];
  pw[0] = 1.0;
  p[0] = 1.0;
  if constexpr (N >= 1) {
    pw[1] = delta;
    p[1] = delta;
  }
#pragma unroll
  for (int m = 2; m < n; ++m) {
    pw[m] = pw[m - 1] * delta;
    p[m] = pw[m] * c_inv_fact[m];
  }
  // alpha' (row sums): Toeplitz(p) * q  +  diag(pw) * Hankel(1/k!) * r
#pragma unroll
  for (int a = 0; a < n; ++a) {
    double acc = q[a];
#pragma unroll
    for (int b = 1; b <= a; ++b) acc = fma(q[a - b], p[b], acc);
    if (a < N) {
      double s = r[1] * c_inv_fact[a + 1];
#pragma unroll
      for (int k = 2; k <= N - a; ++k) s = fma(r[k], c_inv_fact[a + k], s);
      acc = (a == 0) ? acc + s : fma(pw[a], s, acc);
    }
    qo[a] = acc;
  }
  // beta' (column sums): Toeplitz(p) * r (strictly lower) + diag(pw) * Hankel(1/k!) * q
#pragma unroll
  for (int b = 0; b < n; ++b) {
    double t = (b <= 1) ? q[0] : q[0] * c_inv_fact[b];
#pragma unroll
    for (int k = 1; k <= N - b; ++k) t = fma(q[k], c_inv_fact[b + k], t);
    if (b == 0) {
      ro[0] = t;
    } else {
      double acc = r[b];
#pragma unroll
      for (int a = 1; a < b; ++a) acc = fma(r[b - a], p[a], acc);
      ro[b] = fma(pw[b], t, acc);
    }
  }
  if constexpr (N >= 1) {
    if (fault) {
      const double c11 = 2.0 * q[0] * delta;
      qo[1] -= c11;
      ro[1] -= c11;
    }
  }
  double total = qo[0];
#pragma unroll
  for (int a = 1; a < n; ++a) total = fma(qo[a], c_inv_fact[a], total);
  return total;
}

// Literal reference tile step (wavefront.cpp:35-59) on UNSCALED series with a
// runtime order: same expression `b * (pw[min(i,j)] * w[i][j])`, row sums over
// j ascending, column sums accumulated over i ascending, total over rows --
// with every product and sum rounded separately (no FMA), so it is
// bit-identical to the reference.  `w` has row stride kMaxOrder + 1.
__device__ __forceinline__ double tile_step_literal(int order, const double* alpha, const double* beta,
                                                    double delta, const double* w, double* out_alpha,
                                                    double* out_beta) {
  const int n = order + 1;
  double pw[kMaxOrder + 1];
  pw[0] = 1.0;
  for (int m = 1; m < n; ++m) pw[m] = __dmul_rn(pw[m - 1], delta);
  for (int j = 0; j < n; ++j) out_beta[j] = 0.0;
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* wrow = w + i * (kMaxOrder + 1);
    double row_sum = 0.0;
    for (int j = 0; j < n; ++j) {
      const double b = (i >= j) ? alpha[i - j] : beta[j - i];
      const double val = __dmul_rn(b, __dmul_rn(pw[i < j ? i : j], wrow[j]));
      row_sum = __dadd_rn(row_sum, val);
      out_beta[j] = __dadd_rn(out_beta[j], val);
    }
    out_alpha[i] = row_sum;
    total = __dadd_rn(total, row_sum);
  }
  return total;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

}  // namespace skb
