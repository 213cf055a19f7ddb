// Auxiliary kernels around the sweep: increments (K1), the order pre-pass
// (per-series increment norms for the Cauchy-Schwarz bound and the exact
// max|rho| scan), knot-grid boundary initialisation, re-sweep bookkeeping and
// single-tile entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

#include "sk_device.cuh"
#include "sk_internal.h"

namespace skb {

// time_series.cpp:32-42: dz_k = z_{k+1} - z_k.  Device layout per series:
// `len` rows of `ld` doubles -- row 0 is zeros, row k+1 holds dz_k, columns
// >= dim are zero -- so the sweep's row -1 reads a zero vector and every
// row is 16-byte aligned for ld even.
__global__ void increments_kernel(const double* __restrict__ v, size_t nseries, size_t len, size_t dim, size_t ld,
                                  double* __restrict__ out) {
  const size_t per = len * ld;
  const size_t total = nseries * per;
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t s = t / per;
    const size_t e = t - s * per;
    const size_t row = e / ld, c = e - row * ld;
    double val = 0.0;
    if (row > 0 && c < dim) {
      const double* src = v + s * len * dim + (row - 1) * dim + c;
      val = src[dim] - src[0];
    }
    out[t] = val;
  }
}

// The same layout for ld = LD in {2, 4, 8, 16} (d <= 16), one thread per
// output row (no index divisions: rows of a series along x, series along y),
// fused with the per-series max_k sum_c dz_k[c]^2 of max_sqnorm_kernel (same
// FMA order, so the same bits) when `sqn` is set.  Row k + 1 reads input rows
// k and k + 1; the neighbour's row comes from L1.
template <int LD>
__global__ void __launch_bounds__(256) increments_rows_kernel(const double* __restrict__ v, size_t nseries, size_t len,
                                                              int dim, double* __restrict__ out,
                                                              unsigned long long* __restrict__ sqn) {
  const size_t row = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const int lane = threadIdx.x & 31;
  for (size_t s = blockIdx.y; s < nseries; s += gridDim.y) {
    double best = 0.0;
    if (row < len) {
      double val[LD];
#pragma unroll
      for (int c = 0; c < LD; ++c) val[c] = 0.0;
      if (row > 0) {
        const double* src = v + (s * len + row - 1) * dim;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < LD; ++c)
          if (c < dim) {
            val[c] = src[dim + c] - src[c];
            acc = fma(val[c], val[c], acc);
          }
        best = acc;
      }
      double2* dst = reinterpret_cast<double2*>(out + (s * len + row) * LD);
#pragma unroll
      for (int c = 0; c < LD; c += 2) dst[c / 2] = make_double2(val[c], val[c + 1]);
    }
    if (sqn) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (lane == 0 && best > 0.0) atomicMax(sqn + s, static_cast<unsigned long long>(__double_as_longlong(best)));
    }
  }
}

// Per series: max_k sum_c dz_k[c]^2 (feeds the Cauchy-Schwarz upper bound of
// max|rho| and the fast-dot error bound of the exact-order path; its rounding
// is covered by their slack).  `bps` blocks per series, rows strided across
// them; out[] holds the bits of a nonnegative double, zeroed by the launcher,
// so atomicMax on the bits is the max of the values.  d <= 16: a thread per
// row, coordinates in order; d > 16: a warp per row, lanes over coordinates
// (coalesced rows of ld doubles).
template <bool WARP_ROW>
__global__ void max_sqnorm_kernel(const double* __restrict__ inc, size_t count, size_t dim, size_t ld, int bps,
                                  unsigned long long* __restrict__ out) {
  const size_t series = blockIdx.x / bps, part = blockIdx.x - series * bps;
  const double* s = inc + series * (count + 1) * ld + ld;
  const int lane = threadIdx.x & 31;
  double best = 0.0;
  if constexpr (WARP_ROW) {
    const size_t wpb = blockDim.x >> 5;
    for (size_t k = part * wpb + (threadIdx.x >> 5); k < count; k += bps * wpb) {
      double acc = 0.0;
      for (size_t c = lane; c < dim; c += 32) acc = fma(s[k * ld + c], s[k * ld + c], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      best = fmax(best, acc);
    }
  } else {
    for (size_t k = part * blockDim.x + threadIdx.x; k < count; k += static_cast<size_t>(bps) * blockDim.x) {
      double acc = 0.0;
      for (size_t c = 0; c < dim; ++c) acc = fma(s[k * ld + c], s[k * ld + c], acc);
      best = fmax(best, acc);
    }
  }
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (threadIdx.x == 0 && best > 0.0) atomicMax(out + series, static_cast<unsigned long long>(__double_as_longlong(best)));
  }
}

// Exact max|rho| per pair (time_series.cpp:64-73): sequential non-FMA dot in
// coordinate order, so the value is bit-identical and estimate_order's
// thresholds cannot flip.  blockIdx.y = launch-local pair; threads own rows.
template <int DP>
__global__ void maxrho_scan_kernel(const double* __restrict__ xinc, const double* __restrict__ yinc,
                                   const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                                   unsigned long long sx, unsigned long long sy, int rows, int cols, int dim, int ld,
                                   unsigned long long* __restrict__ out) {
  const int pr = blockIdx.y;
  const double* xs = xinc + px[pr] * sx + ld;
  const double* ys = yinc + py[pr] * sy + ld;
  double best = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    const double* yr = ys + static_cast<size_t>(i) * ld;
    if constexpr (DP > 0) {
      double yv[DP];
#pragma unroll
      for (int c = 0; c < DP; ++c) yv[c] = (c < dim) ? yr[c] : 0.0;
      for (int j = 0; j < cols; ++j) {
        const double* xr = xs + static_cast<size_t>(j) * ld;
        double xv[DP];
#pragma unroll
        for (int c = 0; c < DP; ++c) xv[c] = (c < dim) ? __ldg(xr + c) : 0.0;
        const double a = fabs(exact_dot<DP>(xv, yv));
        if (best < a) best = a;
      }
    } else {
      for (int j = 0; j < cols; ++j) {
        const double* xr = xs + static_cast<size_t>(j) * ld;
        double acc = __dmul_rn(__ldg(xr), yr[0]);
        for (int c = 1; c < dim; ++c) acc = __dadd_rn(acc, __dmul_rn(__ldg(xr + c), yr[c]));
        const double a = fabs(acc);
        if (best < a) best = a;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best > 0.0)
    atomicMax(out + pr, static_cast<unsigned long long>(__double_as_longlong(best)));
}

// rho table for the large-d path (d > 16) when it fits the memory budget
// (run_sweeps): rho[i][j] = <dy_i, dx_j>, row-major rows x cols per pair; the
// sweep gathers its deltas from it.  Above the budget the sweep's producer
// warps form rho in shared memory instead (sk_sweep.cuh, O(l) memory).
//
// Exact variant: sequential non-FMA dot (bit-identical deltas, needed when
// the caller asks for the exact max|rho|).  One thread per entry.
__global__ void rho_table_exact_kernel(const double* __restrict__ xinc, const double* __restrict__ yinc,
                                       const uint32_t* __restrict__ px, const uint32_t* __restrict__ py,
                                       unsigned long long sx, unsigned long long sy, int rows, int cols, int dim,
                                       int ld, double* __restrict__ tab, unsigned long long tab_stride) {
  const int pr = blockIdx.z;
  const int j = blockIdx.x * 32 + threadIdx.x;
  const int i = blockIdx.y * 8 + threadIdx.y;
  if (i >= rows || j >= cols) return;
  const double* xr = xinc + px[pr] * sx + static_cast<size_t>(j + 1) * ld;
  const double* yr = yinc + py[pr] * sy + static_cast<size_t>(i + 1) * ld;
  double acc = __dmul_rn(__ldg(xr), __ldg(yr));
  for (int c = 1; c < dim; ++c) acc = __dadd_rn(acc, __dmul_rn(__ldg(xr + c), __ldg(yr + c)));
  tab[pr * tab_stride + static_cast<size_t>(i) * cols + j] = acc;
}

// Tensor-core variant: FP64 DMMA (mma.sync m8n8k4 f64) tiled GEMM,
// rho = dY * dX^T.  CTA tile 64 x 64 (i x j), 4 warps of 32 x 32, k staged
// through shared memory in chunks of 32 with cp.async double buffering.
// Increments are zero-padded to ld (multiple of 4), so k-padding is exact.
// GK = k chunk: 32 alone (74 KB of shared memory, 3 CTAs per SM), 16 when the
// GEMM runs beside a latency-bound sweep (41 KB: two fit next to a sweep CTA).
// rowdone (optional): per pair and 64-row block, the number of column blocks
// written -- the sweep's bands start on their rows as soon as they are done.
constexpr int kGT = 64;            // CTA tile edge
template <int GK>
constexpr int gemm_smem() {
  return 2 * 2 * kGT * (GK + 4) * 8;  // [buf][A|B][kGT][GK + 4]: conflict-free fragment loads
}

#ifndef SK_OVERLAP_GK
#define SK_OVERLAP_GK 16
#endif
constexpr int kOverlapGK = SK_OVERLAP_GK;

template <int GK>
__global__ void __launch_bounds__(128) rho_gemm_kernel(const double* __restrict__ xinc,
                                                       const double* __restrict__ yinc,
                                                       const uint32_t* __restrict__ px,
                                                       const uint32_t* __restrict__ py, unsigned long long sx,
                                                       unsigned long long sy, int rows, int cols, int ld,
                                                       double* __restrict__ tab, unsigned long long tab_stride,
                                                       unsigned* __restrict__ rowdone) {
  constexpr int kGK = GK;
  constexpr int kGS = GK + 4;
  extern __shared__ __align__(16) double gsm[];  // [buf][A|B][kGT][kGS]
  const int pr = blockIdx.z;
  const int i0 = blockIdx.y * kGT, j0 = blockIdx.x * kGT;
  const double* ys = yinc + py[pr] * sy + ld;  // row i at ys + i * ld
  const double* xs = xinc + px[pr] * sx + ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto load = [&](int buf, int k0) {
    double* A = gsm + (buf * 2 + 0) * kGT * kGS;
    double* B = gsm + (buf * 2 + 1) * kGT * kGS;
    for (int e = tid; e < kGT * (kGK / 2); e += 128) {
      const int r = e / (kGK / 2), c = (e % (kGK / 2)) * 2;
      const int k = k0 + c;
      const int ia = i0 + r, jb = j0 + r;
      const bool oka = ia < rows && k < ld, okb = jb < cols && k < ld;
      cp_async_16_zfill(A + r * kGS + c, ys + static_cast<size_t>(oka ? ia : 0) * ld + (oka ? k : 0), oka);
      cp_async_16_zfill(B + r * kGS + c, xs + static_cast<size_t>(okb ? jb : 0) * ld + (okb ? k : 0), okb);
    }
    cp_async_commit();
  };

  const int nk = (ld + kGK - 1) / kGK;
  load(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    const int buf = kc & 1;
    if (kc + 1 < nk) {
      load(buf ^ 1, (kc + 1) * kGK);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* A = gsm + (buf * 2 + 0) * kGT * kGS + (wm * 32 + (lane >> 2)) * kGS + (lane & 3);
    const double* B = gsm + (buf * 2 + 1) * kGT * kGS + (wn * 32 + (lane >> 2)) * kGS + (lane & 3);
#pragma unroll
    for (int k4 = 0; k4 < kGK; k4 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = A[t * 8 * kGS + k4];
        b[t] = B[t * 8 * kGS + k4];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_884(acc[mt][nt], a[mt], b[nt]);
    }
    __syncthreads();
  }
  double* out = tab + pr * tab_stride;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int i = i0 + wm * 32 + mt * 8 + (lane >> 2);
    if (i >= rows) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int j = j0 + wn * 32 + nt * 8 + 2 * (lane & 3);
      if (j < cols) out[static_cast<size_t>(i) * cols + j] = acc[mt][nt][0];
      if (j + 1 < cols) out[static_cast<size_t>(i) * cols + j + 1] = acc[mt][nt][1];
    }
  }
  if (rowdone != nullptr) {
    // every thread's tile stores, then one gpu-scope fence and count
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(rowdone + static_cast<size_t>(pr) * gridDim.y + blockIdx.y, 1u);
    }
  }
}

// Knot grid boundary (wavefront.cpp:92-98): K = 1 on a = 0 and b = 0.
__global__ void grid_init_kernel(double* grid, size_t nout, size_t lx, size_t ly) {
  const size_t per = lx * ly;
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < nout * per;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t e = t % per;
    const size_t a = e / ly, b = e - a * ly;
    if (a == 0 || b == 0) grid[t] = 1.0;
  }
}

// step_tile with the reference's exact arithmetic (one thread).
// io: in = alpha[65] | beta[65]; out = alpha'[65] | beta'[65] | total
__global__ void step_tile_literal_kernel(double delta, int order, const double* __restrict__ w65,
                                         const double* __restrict__ in, double* __restrict__ out) {
  double a[kMaxOrder + 1], b[kMaxOrder + 1], oa[kMaxOrder + 1], ob[kMaxOrder + 1];
  for (int m = 0; m <= order; ++m) {
    a[m] = in[m];
    b[m] = in[kMaxOrder + 1 + m];
  }
  const double total = tile_step_literal(order, a, b, delta, w65, oa, ob);
  for (int m = 0; m <= order; ++m) {
    out[m] = oa[m];
    out[kMaxOrder + 1 + m] = ob[m];
  }
  out[2 * (kMaxOrder + 1)] = total;
}

template <int N>
__global__ void step_tile_fast_kernel(double delta, const double* __restrict__ in, double* __restrict__ out) {
  double q[N + 1], r[N + 1], qo[N + 1], ro[N + 1];
  double f = 1.0;
#pragma unroll
  for (int m = 0; m <= N; ++m) {
    if (m > 0) f *= m;
    q[m] = in[m] * f;
    r[m] = in[kMaxOrder + 1 + m] * f;
  }
  const double total = tile_step_scaled<N>(q, r, delta, qo, ro, false);
#pragma unroll
  for (int m = 0; m <= N; ++m) {
    out[m] = qo[m] * c_inv_fact[m];
    out[kMaxOrder + 1 + m] = ro[m] * c_inv_fact[m];
  }
  out[2 * (kMaxOrder + 1)] = total;
}

// Re-sweep bookkeeping (recheck_failures): reset the listed output slots'
// error keys, and gather (value bits, error key) of the listed slots into one
// contiguous buffer [values | keys] for a single device-to-host copy.
__global__ void reset_slots_kernel(const uint32_t* __restrict__ idx, size_t n, unsigned long long* __restrict__ err) {
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<size_t>(gridDim.x) * blockDim.x)
    err[idx[t]] = ~0ull;
}
__global__ void gather_slots_kernel(const uint32_t* __restrict__ idx, size_t n, const double* __restrict__ values,
                                    const unsigned long long* __restrict__ err, unsigned long long* __restrict__ out) {
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    out[t] = static_cast<unsigned long long>(__double_as_longlong(values[idx[t]]));
    out[n + t] = err[idx[t]];
  }
}

// sk_gram_device: launch slot t (pair (pi[t], pj[t])) into both mirrored cells
// of the m x m matrix; a failed entry (error key set) is NaN (gram.cpp:74-77)
__global__ void scatter_gram_kernel(const uint32_t* __restrict__ pi, const uint32_t* __restrict__ pj, size_t n,
                                    size_t m, const double* __restrict__ values,
                                    const unsigned long long* __restrict__ err, double* __restrict__ mat) {
  for (size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double v = err[t] == ~0ull ? values[t] : __longlong_as_double(0x7ff8000000000000ll);
    mat[static_cast<size_t>(pi[t]) * m + pj[t]] = v;
    mat[static_cast<size_t>(pj[t]) * m + pi[t]] = v;
  }
}

// ------------------------------------------------------------- launchers
static int grid_for(size_t work, int threads) {
  size_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g);
}

cudaError_t launch_increments(const double* v, size_t nseries, size_t len, size_t dim, size_t ld, double* out,
                              cudaStream_t st, double* sqn) {
  const size_t work = nseries * len * ld;
  if (work == 0) return cudaSuccess;
  if (sqn) {
    cudaError_t e = cudaMemsetAsync(sqn, 0, nseries * sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  if (ld == 2 || ld == 4 || ld == 8 || ld == 16) {
    const dim3 grid(static_cast<unsigned>((len + 255) / 256), static_cast<unsigned>(std::min<size_t>(nseries, 65535)));
    auto* bits = reinterpret_cast<unsigned long long*>(sqn);
    const int d = static_cast<int>(dim);
    switch (ld) {
      case 2: increments_rows_kernel<2><<<grid, 256, 0, st>>>(v, nseries, len, d, out, bits); break;
      case 4: increments_rows_kernel<4><<<grid, 256, 0, st>>>(v, nseries, len, d, out, bits); break;
      case 8: increments_rows_kernel<8><<<grid, 256, 0, st>>>(v, nseries, len, d, out, bits); break;
      default: increments_rows_kernel<16><<<grid, 256, 0, st>>>(v, nseries, len, d, out, bits); break;
    }
    return cudaGetLastError();
  }
  increments_kernel<<<grid_for(work, 256), 256, 0, st>>>(v, nseries, len, dim, ld, out);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess || !sqn) return e;
  return launch_max_sqnorm(out, nseries, len - 1, dim, ld, sqn, st);
}

cudaError_t launch_max_sqnorm(const double* inc, size_t nseries, size_t count, size_t dim, size_t ld, double* out,
                              cudaStream_t st) {
  if (nseries == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(out, 0, nseries * sizeof(double), st);
  if (e != cudaSuccess) return e;
  const bool warp_row = dim > 16;
  const size_t rows_per_block = warp_row ? 8 : 256;
  const size_t want = (count + rows_per_block - 1) / rows_per_block;
  const size_t cap = std::max<size_t>(1, 148 * 16 / nseries);
  const int bps = static_cast<int>(std::max<size_t>(1, std::min(want, cap)));
  const unsigned blocks = static_cast<unsigned>(nseries * bps);
  auto* bits = reinterpret_cast<unsigned long long*>(out);
  if (warp_row)
    max_sqnorm_kernel<true><<<blocks, 256, 0, st>>>(inc, count, dim, ld, bps, bits);
  else
    max_sqnorm_kernel<false><<<blocks, 256, 0, st>>>(inc, count, dim, ld, bps, bits);
  return cudaGetLastError();
}

cudaError_t launch_maxrho_scan(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                               size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                               int dim, int ld, unsigned long long* out, cudaStream_t st) {
  if (npairs == 0) return cudaSuccess;
  const int threads = 128;
  const int bx = (rows + threads - 1) / threads;
  const dim3 grid(bx, static_cast<unsigned>(npairs));
  const int dp = pick_dp(dim);
  switch (dp) {
    case 2: maxrho_scan_kernel<2><<<grid, threads, 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, out); break;
    case 4: maxrho_scan_kernel<4><<<grid, threads, 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, out); break;
    case 8: maxrho_scan_kernel<8><<<grid, threads, 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, out); break;
    case 16: maxrho_scan_kernel<16><<<grid, threads, 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, out); break;
    default: maxrho_scan_kernel<0><<<grid, threads, 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, out); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rho_table(const double* xinc, const double* yinc, const uint32_t* px, const uint32_t* py,
                             size_t npairs, unsigned long long sx, unsigned long long sy, int rows, int cols,
                             int dim, int ld, bool exact, double* tab, unsigned long long tab_stride,
                             cudaStream_t st, unsigned* rowdone) {
  if (npairs == 0) return cudaSuccess;
  if (exact) {
    const dim3 grid((cols + 31) / 32, (rows + 7) / 8, static_cast<unsigned>(npairs));
    rho_table_exact_kernel<<<grid, dim3(32, 8), 0, st>>>(xinc, yinc, px, py, sx, sy, rows, cols, dim, ld, tab,
                                                         tab_stride);
    return cudaGetLastError();
  }
  // function attributes are per device: set once on each device used
  static std::atomic<unsigned long long> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(rho_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem<32>());
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(rho_gemm_kernel<kOverlapGK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             gemm_smem<kOverlapGK>());
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  const dim3 grid((cols + kGT - 1) / kGT, (rows + kGT - 1) / kGT, static_cast<unsigned>(npairs));
  if (rowdone != nullptr)
    rho_gemm_kernel<kOverlapGK><<<grid, 128, gemm_smem<kOverlapGK>(), st>>>(xinc, yinc, px, py, sx, sy, rows, cols,
                                                                            ld, tab, tab_stride, rowdone);
  else
    rho_gemm_kernel<32><<<grid, 128, gemm_smem<32>(), st>>>(xinc, yinc, px, py, sx, sy, rows, cols, ld, tab,
                                                            tab_stride, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_reset_slots(const uint32_t* idx, size_t n, unsigned long long* err, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  reset_slots_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx, n, err);
  return cudaGetLastError();
}

cudaError_t launch_gather_slots(const uint32_t* idx, size_t n, const double* values, const unsigned long long* err,
                                unsigned long long* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  gather_slots_kernel<<<grid_for(n, 256), 256, 0, st>>>(idx, n, values, err, out);
  return cudaGetLastError();
}

cudaError_t launch_scatter_gram(const uint32_t* pi, const uint32_t* pj, size_t n, size_t m, const double* values,
                                const unsigned long long* err, double* mat, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  scatter_gram_kernel<<<grid_for(n, 256), 256, 0, st>>>(pi, pj, n, m, values, err, mat);
  return cudaGetLastError();
}

cudaError_t launch_grid_init(double* grid, size_t nout, size_t lx, size_t ly, cudaStream_t st) {
  const size_t work = nout * lx * ly;
  if (work == 0) return cudaSuccess;
  grid_init_kernel<<<grid_for(work, 256), 256, 0, st>>>(grid, nout, lx, ly);
  return cudaGetLastError();
}

cudaError_t launch_step_tile_literal(double delta, int order, const double* w65, const double* in, double* out,
                                     cudaStream_t st) {
  step_tile_literal_kernel<<<1, 1, 0, st>>>(delta, order, w65, in, out);
  return cudaGetLastError();
}

cudaError_t launch_step_tile_fast(double delta, int order, const double* in, double* out, cudaStream_t st) {
  switch (order) {
#define SK_FAST_CASE(NN) \
  case NN: step_tile_fast_kernel<NN><<<1, 1, 0, st>>>(delta, in, out); break;
    SK_FAST_CASE(1) SK_FAST_CASE(2) SK_FAST_CASE(3) SK_FAST_CASE(4) SK_FAST_CASE(5) SK_FAST_CASE(6)
    SK_FAST_CASE(7) SK_FAST_CASE(8) SK_FAST_CASE(9) SK_FAST_CASE(10) SK_FAST_CASE(11) SK_FAST_CASE(12)
    SK_FAST_CASE(13) SK_FAST_CASE(14) SK_FAST_CASE(15) SK_FAST_CASE(16)
#undef SK_FAST_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace skb
