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
//   * alpha (bottom-edge series) moves one lane up per step by one rotation
//     shuffle; lane 31, whose alpha' has just been handed to the band above,
//     carries lane 0's input (the band-below alpha of column s) into it;
//   * the band-below alpha arrives through a per-pair column buffer in
//     global memory (L2-resident), published every kPublish columns with
//     st.release and staged kChunk columns ahead into shared memory with
//     ld.acquire + cp.async;
//   * the column increments dx_j stream through a per-warp shared-memory ring
//     (cp.async, one chunk ahead, bank-conflict-free padded rows); dy_i stays
//     in registers.
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

constexpr int kChunk = 16;        // columns per staging group
constexpr int kPublish = 32;      // columns per progress publication
constexpr int kRing = 64;         // dx ring rows (>= 2 kChunk + 32)
#ifndef SK_SWEEP_WARPS
#define SK_SWEEP_WARPS 1
#endif
// Warps per CTA.  Warps are fully independent; one-warp CTAs avoid losing
// residency to CTA-granular register allocation.
constexpr int kSweepWarps = SK_SWEEP_WARPS;
#ifndef SK_MIN_BLOCKS
#define SK_MIN_BLOCKS 1
#endif

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
  int dim, order;                 // dim: logical d (row stride of the increments is DP)
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

__host__ __device__ constexpr int series_len(int N) { return N > 0 ? N + 1 : kMaxOrder + 1; }
__host__ __device__ constexpr int col_stride(int N) { return (series_len(N) + 1) & ~1; }
// dx ring row stride in doubles: 16-byte rows padded so that the 8 lanes of
// an LDS.128 phase (columns j, j-1, ..., j-7) hit distinct bank groups.
__host__ __device__ constexpr int ring_stride(int DP) { return DP <= 2 ? 2 : DP + 2; }
// per warp: alpha stage (2 groups) | dx ring (DP > 0) | delta stage
// (1 group computed in place for DP > 0, 2 groups copied from the table for DP = 0)
__host__ __device__ constexpr int stage_doubles_per_warp(int N, int DP) {
  return 2 * kChunk * col_stride(N) + (DP > 0 ? kRing * ring_stride(DP) + kChunk * 32 : 2 * kChunk * 32);
}

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
// EXACT: delta by the reference's sequential non-FMA dot (bit-identical) and
// per-pair max|delta| tracking (needed when the caller asks for max|rho|).
// EXTRAS: knot-grid / diagonal outputs (propagate_grid, prefix knots).
template <int N, int DP, bool EXACT, bool EXTRAS>
__device__ __forceinline__ void sweep_band(const SweepParams& P, unsigned p, unsigned b, int lane,
                                           double* __restrict__ smem) {
  constexpr int NA = series_len(N);
  constexpr int NP = col_stride(N);
  constexpr int XS = ring_stride(DP);
  constexpr int kStage = kChunk * NP;
  double* s_alpha = smem;                                         // 2 x kChunk x NP
  double* s_ring = smem + 2 * kStage;                             // kRing x XS (DP > 0)
  double* s_delta = s_ring + (DP > 0 ? kRing * XS : 0);           // kChunk x 32 (x2 for DP = 0)
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
    unsigned long long seen0 = 0;
    wait_progress(prog_row + (P.bands - 1),
                  static_cast<unsigned long long>(p - P.slots) * (cols + 1) + cols, seen0);
  }

  // Row increment (register resident for the whole band); increments are
  // stored with row stride DP behind one leading zero row.
  double dy[DP > 0 ? DP : 1];
  const double* xser = nullptr;
  const double* tab = nullptr;
  if constexpr (DP > 0) {
    const double* yrow = P.yinc + P.pair_y[p] * P.sy + static_cast<size_t>(row_ok ? i + 1 : 0) * DP;
#pragma unroll
    for (int c = 0; c < DP; c += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(yrow + c));
      dy[c] = v.x;
      dy[c + 1] = v.y;
    }
    xser = P.xinc + P.pair_x[p] * P.sx + DP;  // row j of the pair at xser + j * DP
  } else {
    tab = P.rho_tab + static_cast<size_t>(p) * P.tab_stride + static_cast<size_t>(b) * (cols + 31) * 32;
    dy[0] = 0.0;
  }

  // Loop-carried state, ping-ponged between the A and B sets so the
  // (unrolled-by-2) step loop needs no register copies:
  //   qo*: this lane's alpha' (lane 31: the feed for lane 0)
  //   ro*: this lane's beta' = beta of the next column of its row.
  // Before a lane's first column (j < 0) it runs the delta = 0 tile on unit
  // series, whose output is the unit series again, so beta is e0 exactly at
  // j = 0 without a select.
  double qoA[NA], roA[NA], qoB[NA], roB[NA];
#pragma unroll
  for (int m = 0; m < NA; ++m) {
    qoA[m] = (m == 0) ? 1.0 : 0.0;
    roA[m] = (m == 0) ? 1.0 : 0.0;
  }
  double mx = 0.0;
  unsigned long long errkey = ~0ull;
  unsigned long long seen = 0;
  const int steps = cols + rb - 1;

  // ---- staging: group g = steps/columns [g K, g K + K): band-below alpha
  // (2 buffers), dx (ring row = column mod kRing) or, on the table path, the
  // deltas of those steps (2 buffers); one cp.async group per g.
  auto stage_group = [&](int g) {
    const int col0 = g * kChunk;
    const int ncol = max(0, min(kChunk, cols - col0));
    if (has_below) {
      const double* src = colbuf + static_cast<size_t>(col0) * NP;
      double* dst = s_alpha + (g & 1) * kStage;
      const int pieces = ncol * NP / 2;
      for (int k = lane; k < pieces; k += 32) cp_async_16(dst + 2 * k, src + 2 * k);
    }
    if constexpr (DP > 0) {
      constexpr int PR = DP / 2;  // 16-byte pieces per dx row
      const int pieces = ncol * PR;
      for (int k = lane; k < pieces; k += 32) {
        const int c = k / PR, part = k - c * PR;
        const int col = col0 + c;
        cp_async_16(s_ring + (col & (kRing - 1)) * XS + 2 * part, xser + static_cast<size_t>(col) * DP + 2 * part);
      }
    } else {
      const int nst = max(0, min(kChunk, steps - col0));
      const double* src = tab + static_cast<size_t>(col0) * 32;
      double* dst = s_delta + (g & 1) * kChunk * 32;
      for (int k = lane; k < nst * 16; k += 32) cp_async_16(dst + 2 * k, src + 2 * k);
    }
    cp_async_commit();
  };
  if (!has_below) {
    // band 0: the bottom edge of the domain is the unit series in every column
    for (int e = lane; e < 2 * kStage; e += 32) s_alpha[e] = (e % NP == 0) ? 1.0 : 0.0;
  }
  if constexpr (DP > 0) {
    // columns -32..-1 (ring rows 32..63): zero increments => delta = 0
    for (int e = lane; e < 32 * XS; e += 32) s_ring[32 * XS + e] = 0.0;
  }
  __syncwarp();
  if (has_below) wait_progress(prog_row + (b - 1), base + min(cols, kChunk), seen);
  stage_group(0);

  const int src_lane = (lane + 31) & 31;
  const bool feeder = lane == 31;
  const double* xw = s_ring;

  // one tile step: column j = s - lane of row i (one basic block: all
  // conditional work is predicated)
  auto step = [&](int s, const double* stage_col, double delta, double (&qo_in)[NA], double (&r_in)[NA],
                  double (&qo_out)[NA], double (&ro_out)[NA]) {
    const int j = s - lane;
    // lane 31's alpha' went to the band above at the end of the previous
    // step; it now carries lane 0's input (predicated shared loads)
#pragma unroll
    for (int m = 0; m < NA; m += 2)
      if (N > 0 || m < n) {
        if (m + 1 < NA)
          ld_shared2_if(feeder, stage_col + m, qo_in[m], qo_in[m + 1]);
        else
          ld_shared_if(feeder, stage_col + m, qo_in[m]);
      }
    double q[NA];
#pragma unroll
    for (int m = 0; m < NA; ++m)
      if (N > 0 || m < n) q[m] = __shfl_sync(0xffffffffu, qo_in[m], src_lane);

    double total;
    if constexpr (N > 0) {
      total = tile_step_scaled<N>(q, r_in, delta, qo_out, ro_out, fault);
    } else {
      total = tile_step_literal(P.order, q, r_in, delta, P.w65, qo_out, ro_out);
    }

    const bool active = row_ok && j >= 0 && j < cols;
    const double ad = fabs(delta);
    if constexpr (EXACT) mx = fmax(mx, active ? ad : 0.0);
    // the reference's throw order inside a tile: delta guard, corner check,
    // non-finite total (wavefront.cpp:150-173); first tile in (diagonal, row)
    // order wins -> per-lane running min of the key, one atomic per band
    const unsigned code = !(ad <= kDeltaOverflowLimit)                   ? kErrDelta
                          : (strict && corner_mismatch(q[0], r_in[0]))   ? kErrCorner
                          : !isfinite(total)                             ? kErrNonFinite
                                                                         : 0u;
    const unsigned long long key = err_key(i, j, code);
    errkey = (active && code != 0u && key < errkey) ? key : errkey;
    st_global_if(active && i == rows - 1 && j == cols - 1, P.values + out, total);
    if constexpr (EXTRAS) {
      if (P.grid)
        st_global_if(active, P.grid + out * P.grid_stride + static_cast<size_t>(j + 1) * (rows + 1) + (i + 1), total);
      if (P.diag) st_global_if(active && i == j, P.diag + out * P.diag_stride + i, total);
    }
    // hand alpha' up to the band above (predicated, lane 31 only)
    const bool hand = has_above && feeder && j >= 0 && j < cols;
    double* dst = colbuf + static_cast<ptrdiff_t>(j) * NP;
#pragma unroll
    for (int m = 0; m < NA; m += 2)
      if (N > 0 || m < n) st_global_cg2_if(hand, dst + m, qo_out[m], (m + 1 < NA) ? qo_out[m + 1] : 0.0);
    st_release_gpu_if(hand && ((((j + 1) % kPublish) == 0) || j + 1 == cols), prog_row + b, base + j + 1);
  };

  const int ngroups_in = (cols + kChunk - 1) / kChunk;
  const int ngroups = DP > 0 ? ngroups_in : (steps + kChunk - 1) / kChunk;
  for (int c0 = 0, chunk = 0; c0 < steps; c0 += kChunk, ++chunk) {
    __syncwarp();  // everyone is done with the buffers group chunk + 1 overwrites
    if (chunk + 1 < ngroups) {
      if (has_below) wait_progress(prog_row + (b - 1), base + min(cols, (chunk + 2) * kChunk), seen);
      stage_group(chunk + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const double* stage = s_alpha + (chunk & 1) * kStage;
    const double* dst = s_delta + (DP > 0 ? 0 : (chunk & 1) * kChunk * 32);
    if constexpr (DP > 0) {
      // the chunk's increment products: 16 independent dots per lane
      // (lane t, step c0 + k -> column c0 + k - t), staged in shared memory
#pragma unroll 4
      for (int k = 0; k < kChunk; ++k) {
        const double* xr = xw + ((c0 + k - lane) & (kRing - 1)) * XS;
        double dx[DP];
#pragma unroll
        for (int c = 0; c < DP; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(xr + c);
          dx[c] = v.x;
          dx[c + 1] = v.y;
        }
        double dl;
        if constexpr (EXACT) {
          dl = exact_dot<DP>(dx, dy);
        } else {
          // pairwise-tree FMA dot (short dependency chain)
          double acc[2] = {dx[0] * dy[0], dx[1] * dy[1]};
#pragma unroll
          for (int c = 2; c < DP; ++c) acc[c & 1] = fma(dx[c], dy[c], acc[c & 1]);
          dl = acc[0] + acc[1];
        }
        s_delta[k * 32 + lane] = dl;
      }
      __syncwarp();
    }
    const int kend = min(kChunk, steps - c0);
    int k = 0;
#pragma unroll 1
    for (; k + 1 < kend; k += 2) {
      const double d0 = dst[k * 32 + lane];
      const double d1 = dst[(k + 1) * 32 + lane];
      step(c0 + k, stage + k * NP, d0, qoA, roA, qoB, roB);
      step(c0 + k + 1, stage + (k + 1) * NP, d1, qoB, roB, qoA, roA);
    }
    if (k < kend) {
      step(c0 + k, stage + k * NP, dst[k * 32 + lane], qoA, roA, qoB, roB);
#pragma unroll
      for (int m = 0; m < NA; ++m) {
        qoA[m] = qoB[m];
        roA[m] = roB[m];
      }
    }
  }
  if (errkey != ~0ull) atomicMin(P.err + out, errkey);
  if constexpr (EXACT) {
    if (P.maxrho) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0 && mx > 0.0)
        atomicMax(P.maxrho + out, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
}

// Persistent: grid = resident CTAs; dynamic shared memory =
// kSweepWarps * stage_doubles_per_warp(N, DP) doubles.
template <int N, int DP, bool EXACT, bool EXTRAS>
__global__ void __launch_bounds__(kSweepWarps * 32, SK_MIN_BLOCKS) sweep_kernel(const SweepParams P) {
  extern __shared__ __align__(16) double s_dyn[];
  double* smem = s_dyn + (threadIdx.x >> 5) * stage_doubles_per_warp(N, DP);
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
    sweep_band<N, DP, EXACT, EXTRAS>(P, p, b, lane, smem);
  }
}

}  // namespace skb
