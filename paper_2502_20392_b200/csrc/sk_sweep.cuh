// Banded systolic wavefront sweep (replaces wavefront.cpp:70-192 `run()` and
// the per-diagonal ThreadPool barrier, thread_pool.cpp:59-85).
//
// Work decomposition
// ------------------
// A pair has rows x cols tiles (rows = ly-1 along the second series y, cols =
// lx-1 along the first series x).  Rows are cut into BANDS of 32; one warp
// sweeps one band (a "unit" = (pair, band)).  Lane t owns tile row
// i = 32 b + t and processes column j = s - t at step s, so the 32 lanes walk
// a skewed anti-diagonal of the band:
//   * beta (left-edge series) of row i stays in lane t's REGISTERS from one
//     column to the next;
//   * alpha (bottom-edge series) moves one lane up per step by warp shuffle;
//   * lane 0 takes alpha from the band below and lane 31 hands its alpha' to
//     the band above through a per-pair column buffer in global memory
//     (L2-resident), published every kChunk columns with st.release and
//     consumed with ld.acquire + cp.async into shared memory.
// No grid-wide barrier and no launch per diagonal exists: dependencies are
// point-to-point progress counters, and every warp of a persistent grid pulls
// units from one atomic queue in an order (group, band, pair-in-group) fixed
// by the host.  A unit only ever waits on units earlier in that order, which
// were handed to running warps, so the schedule cannot deadlock.
//
// Memory: per pair one column buffer cols x NP doubles (NP = N+1 rounded up
// to even) -- O(ell N), the reference's memory contract (wavefront.cpp:100-105).
#pragma once

#include <cstdint>

#include "sk_device.cuh"

namespace skb {

constexpr int kChunk = 16;        // columns per progress publication / alpha stage
constexpr int kSweepWarps = 4;    // warps per CTA (CTAs are independent)

struct SweepParams {
  const double* xinc;             // increments of the column series (first series, x)
  const double* yinc;             // increments of the row series (second series, y)
  const uint32_t* pair_x;         // launch-local pair -> x series index
  const uint32_t* pair_y;         // launch-local pair -> y series index
  const uint32_t* pair_out;       // launch-local pair -> output slot
  unsigned long long sx, sy;      // elements between consecutive series
  const double* w65;              // N == 0: W table, row stride 65 (device memory)
  const double* rho_tab;          // DP == 0: skewed delta table per launch-local pair
  unsigned long long tab_stride;  // elements per pair in rho_tab
  int dim, order;
  int rows, cols, bands, npairs, group, slots;
  unsigned flags;
  double* abuf;                   // slots x cols x NP
  unsigned long long* prog;       // slots x bands progress counters
  unsigned* queue;                // unit counter
  double* values;                 // per output slot: K(1,1)
  unsigned long long* err;        // per output slot: min error key (init ~0)
  unsigned long long* maxrho;     // per output slot: max |delta| bits (init 0) or null
  double* grid;                   // per output slot: lx x ly knot grid, or null
  double* diag;                   // per output slot: K at tiles (i, i), or null
  unsigned long long grid_stride, diag_stride;
};

constexpr unsigned kFlagStrictCorner = 1u;
constexpr unsigned kFlagWFault = 4u;

__device__ __forceinline__ void wait_progress(const unsigned long long* ptr, unsigned long long need,
                                              unsigned long long& seen) {
  // every lane polls the same word (one transaction); acquire orders the
  // lane's later loads of the column buffer after the producer's release.
  if (seen >= need) return;
  unsigned long long v = ld_acquire_gpu(ptr);
  while (v < need) {
    __nanosleep(64);
    v = ld_acquire_gpu(ptr);
  }
  seen = v;
}

// N > 0: register kernel on factorial-scaled series.  N == 0: literal
// reference arithmetic with runtime order P.order (bit-identical tile math,
// series in local memory) for orders above kMaxRegOrder.
template <int N, int DP>
__device__ __forceinline__ void sweep_band(const SweepParams& P, unsigned p, unsigned b, int lane,
                                           double* __restrict__ s_stage /* 2 * kChunk * NP */) {
  constexpr int NA = N > 0 ? N + 1 : kMaxOrder + 1;  // series array length
  constexpr int NP = (NA + 1) & ~1;                   // column-buffer stride (16B aligned)
  const int n = N > 0 ? N + 1 : P.order + 1;
  const int rows = P.rows, cols = P.cols;
  const int row0 = static_cast<int>(b) * 32;
  const int rb = min(32, rows - row0);
  const int i = row0 + lane;
  const bool row_ok = lane < rb;
  const unsigned slot = p % static_cast<unsigned>(P.slots);
  const unsigned long long base = static_cast<unsigned long long>(p) * static_cast<unsigned long long>(cols + 1);
  double* colbuf = P.abuf + static_cast<size_t>(slot) * static_cast<size_t>(cols) * NP;
  unsigned long long* prog_row = P.prog + static_cast<size_t>(slot) * P.bands;
  const bool has_below = b > 0;
  const bool has_above = b + 1 < static_cast<unsigned>(P.bands);
  const unsigned out = P.pair_out[p];
  const bool strict = (P.flags & kFlagStrictCorner) != 0;
  const bool fault = (P.flags & kFlagWFault) != 0;

  // Slot hand-over: band 0 of pair p rewrites the column buffer that the last
  // band of the slot's previous pair (p - slots) reads.
  if (b == 0 && has_above && p >= static_cast<unsigned>(P.slots)) {
    unsigned long long seen = 0;
    wait_progress(prog_row + (P.bands - 1),
                  static_cast<unsigned long long>(p - P.slots) * (cols + 1) + cols, seen);
  }

  // Row increment (register resident for the whole band).
  double dy[DP > 0 ? DP : 1];
  const double* xser = nullptr;
  const double* tab = nullptr;
  if constexpr (DP > 0) {
    const double* yrow = P.yinc + P.pair_y[p] * P.sy + static_cast<size_t>(min(i, rows - 1)) * P.dim;
#pragma unroll
    for (int c = 0; c < DP; ++c) dy[c] = (row_ok && c < P.dim) ? __ldg(yrow + c) : 0.0;
    xser = P.xinc + P.pair_x[p] * P.sx;
  } else {
    tab = P.rho_tab + static_cast<size_t>(p) * P.tab_stride + static_cast<size_t>(b) * (cols + 31) * 32;
    dy[0] = 0.0;
  }

  double q[NA], r[NA], qo[NA], ro[NA];
#pragma unroll
  for (int m = 0; m < NA; ++m) {
    qo[m] = 0.0;
    ro[m] = (m == 0) ? 1.0 : 0.0;
  }
  double mx = 0.0;
  unsigned long long seen = 0;
  const int nchunks_in = (cols + kChunk - 1) / kChunk;
  constexpr int kStage = kChunk * NP;
  // stage chunk c of the band-below's alpha columns into s_stage[c & 1]
  auto stage_chunk = [&](int c) {
    const int col0 = c * kChunk;
    const int ncol = min(kChunk, cols - col0);
    const double* src = colbuf + static_cast<size_t>(col0) * NP;
    double* dst = s_stage + (c & 1) * kStage;
    const int pieces = ncol * NP / 2;
    for (int k = lane; k < pieces; k += 32) cp_async_16(dst + 2 * k, src + 2 * k);
    cp_async_commit();
  };
  if (has_below) {
    wait_progress(prog_row + (b - 1), base + min(cols, kChunk), seen);
    stage_chunk(0);
  }

  const int steps = cols + rb - 1;
  for (int c0 = 0; c0 < steps; c0 += kChunk) {
    const int chunk = c0 / kChunk;
    if (has_below) {
      __syncwarp();  // lane 0 is done with the buffer chunk + 1 will overwrite
      if (chunk + 1 < nchunks_in) {
        wait_progress(prog_row + (b - 1), base + min(cols, (chunk + 2) * kChunk), seen);
        stage_chunk(chunk + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
    }
    const double* stage = s_stage + (chunk & 1) * kStage;
    const int kend = min(kChunk, steps - c0);
    for (int k = 0; k < kend; ++k) {
      const int s = c0 + k;
      const int j = s - lane;
      const bool active = row_ok && j >= 0 && j < cols;

      // alpha: from the lane below (previous step), lane 0 from the band below
#pragma unroll
      for (int m = 0; m < NA; ++m)
        if (N > 0 || m < n) q[m] = __shfl_up_sync(0xffffffffu, qo[m], 1);
      if (lane == 0) {
        if (has_below) {
          if (s < cols) {
#pragma unroll
            for (int m = 0; m < NA; ++m)
              if (N > 0 || m < n) q[m] = stage[k * NP + m];
          }
        } else {
#pragma unroll
          for (int m = 0; m < NA; ++m) q[m] = (m == 0) ? 1.0 : 0.0;
        }
      }
      // beta: own previous output; the unit series on the domain edge j = 0
#pragma unroll
      for (int m = 0; m < NA; ++m) r[m] = (j == 0) ? (m == 0 ? 1.0 : 0.0) : ro[m];

      // increment product
      double delta;
      if constexpr (DP > 0) {
        const int jc = min(max(j, 0), cols - 1);
        const double* xcol = xser + static_cast<size_t>(jc) * P.dim;
        double dx[DP];
        if (P.dim == DP) {
#pragma unroll
          for (int c = 0; c < DP; c += 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(xcol + c));
            dx[c] = v.x;
            dx[c + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < DP; ++c) dx[c] = (c < P.dim) ? __ldg(xcol + c) : 0.0;
        }
        delta = exact_dot<DP>(dx, dy);
      } else {
        delta = (active) ? tab[static_cast<size_t>(s) * 32 + lane] : 0.0;
      }

      double total;
      if constexpr (N > 0) {
        total = tile_step_scaled<N>(q, r, delta, qo, ro, fault);
      } else {
        total = tile_step_literal(P.order, q, r, delta, P.w65, qo, ro);
      }

      if (active) {
        const double ad = fabs(delta);
        mx = fmax(mx, ad);
        unsigned code = 0;
        if (!(ad <= kDeltaOverflowLimit))
          code = kErrDelta;
        else if (strict && corner_mismatch(q[0], r[0]))
          code = kErrCorner;
        else if (!isfinite(total))
          code = kErrNonFinite;
        if (code) atomicMin(P.err + out, err_key(i, j, code));
        if (P.grid) P.grid[out * P.grid_stride + static_cast<size_t>(j + 1) * (rows + 1) + (i + 1)] = total;
        if (P.diag && i == j) P.diag[out * P.diag_stride + i] = total;
        if (i == rows - 1 && j == cols - 1) P.values[out] = total;
      }
      // hand alpha' up to the band above
      if (has_above && lane == 31 && j >= 0 && j < cols) {
        double* dst = colbuf + static_cast<size_t>(j) * NP;
#pragma unroll
        for (int m = 0; m < NA; m += 2) {
          if (N > 0 || m < n) {
            double2 v;
            v.x = qo[m];
            v.y = (m + 1 < NA) ? qo[m + 1] : 0.0;
            __stcg(reinterpret_cast<double2*>(dst + m), v);
          }
        }
        if (((j + 1) % kChunk) == 0 || j + 1 == cols) st_release_gpu(prog_row + b, base + j + 1);
      }
    }
  }
  if (P.maxrho) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.0) atomicMax(P.maxrho + out, static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}

template <int N>
__host__ __device__ constexpr int stage_doubles_per_warp() {
  return 2 * kChunk * ((((N > 0 ? N + 1 : kMaxOrder + 1)) + 1) & ~1);
}

// Persistent: grid = resident CTAs; dynamic shared memory =
// kSweepWarps * stage_doubles_per_warp<N>() doubles.
template <int N, int DP>
__global__ void __launch_bounds__(kSweepWarps * 32) sweep_kernel(const SweepParams P) {
  extern __shared__ __align__(16) double s_dyn[];
  double* s_stage = s_dyn + (threadIdx.x >> 5) * stage_doubles_per_warp<N>();
  const int lane = threadIdx.x & 31;
  const unsigned total_units = static_cast<unsigned>(P.npairs) * static_cast<unsigned>(P.bands);
  const unsigned gsz = static_cast<unsigned>(P.group) * static_cast<unsigned>(P.bands);
  for (;;) {
    unsigned u = 0;
    if (lane == 0) u = atomicAdd(P.queue, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= total_units) return;
    // unit order: (group g, band b, pair q within the group)
    const unsigned g = u / gsz;
    const unsigned rem = u - g * gsz;
    const unsigned g0 = g * static_cast<unsigned>(P.group);
    const unsigned gcount = min(static_cast<unsigned>(P.group), static_cast<unsigned>(P.npairs) - g0);
    const unsigned b = rem / gcount;
    const unsigned p = g0 + (rem - b * gcount);
    sweep_band<N, DP>(P, p, b, lane, s_stage);
  }
}

}  // namespace skb
