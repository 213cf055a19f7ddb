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
//   * alpha (bottom-edge series) moves one lane up per step through a
//     per-warp shared-memory slot array (lane t reads slot t-1, writes slot
//     t); lane 0 reads the band below's alpha, lane 31 writes into a chunk
//     buffer that the warp hands to the band above once per chunk;
//   * the band-below alpha arrives through a per-pair column buffer in
//     global memory (L2-resident), published every kPublish columns with
//     a fence + st.release and staged one chunk ahead into shared memory with
//     ld.acquire + cp.async;
//   * the column increments dx_j stream through a per-warp shared-memory ring
//     (cp.async, one chunk ahead, bank-conflict-free padded rows); the
//     increment products of a whole chunk are contracted up front (16
//     independent dots per lane) into shared memory.
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
  const double* rho_tab;          // DP == 0: rho table (rows x cols, row-major) per launch-local pair
  unsigned long long tab_stride;  // elements per pair in rho_tab
  int dim, order;                 // dim: logical d (row stride of the increments is DP)
  int rows, cols, bands, npairs, group, slots;
  unsigned flags;
  double* abuf;                   // slots x cols x NP
  unsigned long long* prog;       // slots x bands progress counters
  unsigned* queue;                // unit counter
  unsigned long long* watchdog;   // [0] abort flag, [1..4] first stuck wait (p, b, need, seen)
  unsigned long long watchdog_ns; // give up a dependency wait after this long
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
// per warp: band-below alpha stage (2 groups) | lane-to-lane alpha slots (2 x 32)
// | lane 31's outputs of the chunk | dx ring (DP > 0) | delta stage (1 group
// computed in place for DP > 0, 2 groups copied from the table for DP = 0)
__host__ __device__ constexpr int stage_doubles_per_warp(int N, int DP) {
  return 2 * kChunk * col_stride(N) + 2 * 32 * col_stride(N) + kChunk * col_stride(N) +
         (DP > 0 ? kRing * ring_stride(DP) + kChunk * 32 : 2 * kChunk * 32);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Dependency wait with a watchdog: a wait that exceeds P.watchdog_ns (a
// scheduling bug -- by construction every awaited unit is running) records
// itself, raises the abort flag and returns false instead of hanging the GPU;
// every other waiting warp then bails out too.
static __device__ __noinline__ bool wait_progress_slow(const unsigned long long* ptr, unsigned long long need,
                                                       unsigned long long& seen, unsigned long long* wd,
                                                       unsigned long long limit_ns, unsigned p, unsigned b) {
  // poll with relaxed loads (no L1 invalidation per poll) and a growing
  // back-off; the acquire is taken once the value is there
  const unsigned long long t0 = globaltimer_ns();
  unsigned ns = 32;
  for (unsigned it = 1;; ++it) {
    __nanosleep(ns);
    if (ns < 1024) ns += ns >> 1;
    if (ld_relaxed_gpu(ptr) >= need) break;
    if ((it & 15) == 0) {
      if (*reinterpret_cast<volatile unsigned long long*>(wd) != 0) return false;
      if (globaltimer_ns() - t0 > limit_ns) {
        if ((threadIdx.x & 31) == 0 && atomicCAS(wd, 0ull, 1ull) == 0ull) {
          wd[1] = p;
          wd[2] = b;
          wd[3] = need;
          wd[4] = ld_relaxed_gpu(ptr);
        }
        return false;
      }
    }
  }
  seen = ld_acquire_gpu(ptr);
  return true;
}

__device__ __forceinline__ bool wait_progress(const SweepParams& P, const unsigned long long* ptr,
                                              unsigned long long need, unsigned long long& seen, unsigned p,
                                              unsigned b) {
  if (seen >= need) return true;
  const unsigned long long v = ld_acquire_gpu(ptr);  // every lane polls the same word
  if (v >= need) {
    seen = v;
    return true;
  }
  return wait_progress_slow(ptr, need, seen, P.watchdog, P.watchdog_ns, p, b);
}

template <int NA>
__device__ __forceinline__ void lds_series(const double* src, double (&v)[NA], int n) {
#pragma unroll
  for (int m = 0; m < NA; m += 2) {
    if (m + 1 < NA) {
      if (NA <= kMaxRegOrder + 1 || m < n) {
        const double2 t = *reinterpret_cast<const double2*>(src + m);
        v[m] = t.x;
        v[m + 1] = t.y;
      }
    } else if (NA <= kMaxRegOrder + 1 || m < n) {
      v[m] = src[m];
    }
  }
}

template <int NA>
__device__ __forceinline__ void sts_series(double* dst, const double (&v)[NA], int n) {
#pragma unroll
  for (int m = 0; m < NA; m += 2) {
    if (NA <= kMaxRegOrder + 1 || m < n) {
      double2 t;
      t.x = v[m];
      t.y = (m + 1 < NA) ? v[m + 1] : 0.0;
      *reinterpret_cast<double2*>(dst + m) = t;
    }
  }
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
  double* s_alpha = smem;                                   // 2 x kChunk x NP
  double* s_pass = s_alpha + 2 * kStage;                    // 2 x 32 x NP (step parity)
  double* s_out = s_pass + 64 * NP;                         // kChunk x NP
  double* s_ring = s_out + kStage;                          // kRing x XS (DP > 0)
  double* s_delta = s_ring + (DP > 0 ? kRing * XS : 0);     // kChunk x 32 (x2 for DP = 0)
  const int n = N > 0 ? N + 1 : P.order + 1;
  const int rows = P.rows, cols = P.cols;
  const int row0 = static_cast<int>(b) * 32;
  const int rb = min(32, rows - row0);
  const int i = row0 + lane;
  const bool row_ok = lane < rb;
  const bool last_row = row_ok && i == rows - 1;
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
    if (!wait_progress(P, prog_row + (P.bands - 1),
                       static_cast<unsigned long long>(p - P.slots) * (cols + 1) + cols, seen0, p, b))
      return;
  }

  // increments are stored with row stride DP behind one leading zero row
  const double* yrow = nullptr;
  const double* xser = nullptr;
  const double* tab = nullptr;
  if constexpr (DP > 0) {
    yrow = P.yinc + P.pair_y[p] * P.sy + static_cast<size_t>(row_ok ? i + 1 : 0) * DP;
    xser = P.xinc + P.pair_x[p] * P.sx + DP;  // row j of the pair at xser + j * DP
  } else {
    tab = P.rho_tab + static_cast<size_t>(p) * P.tab_stride;  // rows x cols, row-major
  }

  // Loop-carried register state: this lane's beta (the left edge of its next
  // tile).  Before a lane's first column (j < 0) it runs the delta = 0 tile
  // on unit series, whose output is the unit series again, so beta is e0
  // exactly at j = 0 without a select (the alpha slots start at e0 too).
  double roA[NA], roB[NA];
#pragma unroll
  for (int m = 0; m < NA; ++m) roA[m] = (m == 0) ? 1.0 : 0.0;
  double mx = 0.0;
  unsigned jkey = ~0u;  // (first failing column << 2) | code for this lane
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
      // row-major rho table: lane t gathers rho(i, g K + k - t), k < K,
      // zero-filled outside the pair (8-byte cp.async, consecutive lanes ->
      // consecutive shared words)
      double* dst = s_delta + (g & 1) * kChunk * 32 + lane;
      const double* trow = tab + static_cast<size_t>(row_ok ? i : 0) * cols;
#pragma unroll 4
      for (int k = 0; k < kChunk; ++k) {
        const int j = col0 + k - lane;
        const bool ok = row_ok && j >= 0 && j < cols;
        cp_async_8_zfill(dst + k * 32, trow + (ok ? j : 0), ok);
      }
    }
    cp_async_commit();
  };
  if (!has_below) {
    // band 0: the bottom edge of the domain is the unit series in every column
    for (int e = lane; e < 2 * kStage; e += 32) s_alpha[e] = (e % NP == 0) ? 1.0 : 0.0;
  }
  for (int e = lane; e < 64 * NP; e += 32) s_pass[e] = (e % NP == 0) ? 1.0 : 0.0;
  if constexpr (DP > 0) {
    // columns -32..-1 (ring rows 32..63): zero increments => delta = 0
    for (int e = lane; e < 32 * XS; e += 32) s_ring[32 * XS + e] = 0.0;
  }
  __syncwarp();
  if (has_below && !wait_progress(P, prog_row + (b - 1), base + min(cols, kChunk), seen, p, b)) return;
  stage_group(0);

  // step s writes slot [s & 1][lane] and reads [(s - 1) & 1][lane - 1]: the
  // double buffer needs only one __syncwarp per step (RAW); the WAR reuse
  // two steps later is ordered by the intervening one
  double* const my_pass = s_pass + lane * NP;
  const double* const below_pass = s_pass + (lane - 1) * NP;

  // one tile step: column j = s - lane of row i
  auto step = [&](int s, int k, int par, const double* stage, double delta, double (&r_in)[NA],
                  double (&ro_out)[NA]) {
    const int j = s - lane;
    double q[NA], qo[NA];
    // alpha: lane 0 from the band below (stage), lane t from lane t-1's slot
    lds_series<NA>(lane == 0 ? stage + k * NP : below_pass + (par ^ 1) * 32 * NP, q, n);

    double total;
    if constexpr (N > 0) {
      total = tile_step_scaled<N>(q, r_in, delta, qo, ro_out, fault);
    } else {
      total = tile_step_literal(P.order, q, r_in, delta, P.w65, qo, ro_out);
    }
    // alpha' up: lane 31 parks it for the band above, the others in their slot
    sts_series<NA>(lane == 31 ? s_out + k * NP : my_pass + par * 32 * NP, qo, n);
    __syncwarp();

#ifndef SK_EXPERIMENT_NO_CHECKS
    const bool active = row_ok && j >= 0 && j < cols;
    // the reference's throw order inside a tile: delta guard (checked when
    // the chunk's deltas are formed), corner check, non-finite total
    // (wavefront.cpp:150-173); the first failing tile of the lane wins
    const unsigned code = (strict && corner_mismatch(q[0], r_in[0])) ? kErrCorner
                          : !isfinite(total)                         ? kErrNonFinite
                                                                     : 0u;
    const unsigned kk = (static_cast<unsigned>(j) << 2) | code;
    jkey = (active && code != 0u && kk < jkey) ? kk : jkey;
#else
    const bool active = row_ok && j >= 0 && j < cols;
#endif
    st_global_if(last_row && j == cols - 1, P.values + out, total);
    if constexpr (EXTRAS) {
      if (P.grid)
        st_global_if(active, P.grid + out * P.grid_stride + static_cast<size_t>(j + 1) * (rows + 1) + (i + 1), total);
      if (P.diag) st_global_if(active && i == j, P.diag + out * P.diag_stride + i, total);
    }
  };

  const int ngroups_in = (cols + kChunk - 1) / kChunk;
  const int ngroups = DP > 0 ? ngroups_in : (steps + kChunk - 1) / kChunk;
  for (int c0 = 0, chunk = 0; c0 < steps; c0 += kChunk, ++chunk) {
    __syncwarp();  // everyone is done with the buffers group chunk + 1 overwrites
    if (chunk + 1 < ngroups) {
      if (has_below && !wait_progress(P, prog_row + (b - 1), base + min(cols, (chunk + 2) * kChunk), seen, p, b))
        return;
      stage_group(chunk + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const double* stage = s_alpha + (chunk & 1) * kStage;
    const double* dl = s_delta + (DP > 0 ? 0 : (chunk & 1) * kChunk * 32);
    const int kend = min(kChunk, steps - c0);
    // the chunk's increment products (lane t, step c0 + k -> column c0 + k - t)
    // with the delta guard (wavefront.cpp:150-155) and max|delta|
    {
      double dy[DP > 0 ? DP : 1];
      if constexpr (DP > 0) {
#pragma unroll
        for (int c = 0; c < DP; c += 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(yrow + c));
          dy[c] = v.x;
          dy[c + 1] = v.y;
        }
      }
#pragma unroll 1
      for (int k0 = 0; k0 < kChunk; k0 += 4) {
        double dd[4];
        if constexpr (DP > 0) {
          // four columns at a time: all loads first, then four independent
          // two-accumulator dots
          double dx[4][DP];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* xr = s_ring + ((c0 + k0 + u - lane) & (kRing - 1)) * XS;
#pragma unroll
            for (int c = 0; c < DP; c += 2) {
              const double2 v = *reinterpret_cast<const double2*>(xr + c);
              dx[u][c] = v.x;
              dx[u][c + 1] = v.y;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if constexpr (EXACT) {
              dd[u] = exact_dot<DP>(dx[u], dy);
            } else {
              double e0 = dx[u][0] * dy[0], e1 = dx[u][1] * dy[1];
#pragma unroll
              for (int c = 2; c < DP; c += 2) {
                e0 = fma(dx[u][c], dy[c], e0);
                e1 = fma(dx[u][c + 1], dy[c + 1], e1);
              }
              dd[u] = e0 + e1;
            }
            s_delta[(k0 + u) * 32 + lane] = dd[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) dd[u] = dl[(k0 + u) * 32 + lane];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          const int j = c0 + k - lane;
          const bool act = row_ok && j >= 0 && j < cols && k < kend;
          const double ad = fabs(dd[u]);
          if constexpr (EXACT) mx = fmax(mx, act ? ad : 0.0);
          const unsigned kk = (static_cast<unsigned>(j) << 2) | kErrDelta;
          jkey = (act && !(ad <= kDeltaOverflowLimit) && kk < jkey) ? kk : jkey;
        }
      }
    }
    __syncwarp();
    int k = 0;
#pragma unroll 1
    for (; k + 1 < kend; k += 2) {
      const double d0 = dl[k * 32 + lane];
      const double d1 = dl[(k + 1) * 32 + lane];
      step(c0 + k, k, 0, stage, d0, roA, roB);
      step(c0 + k + 1, k + 1, 1, stage, d1, roB, roA);
    }
    if (k < kend) {
      step(c0 + k, k, k & 1, stage, dl[k * 32 + lane], roA, roB);
#pragma unroll
      for (int m = 0; m < NA; ++m) roA[m] = roB[m];
    }
    // hand lane 31's alpha' of this chunk (columns c0 - 31 .. c0 + kend - 32)
    // to the band above, then publish progress every kPublish columns
    if (has_above) {
      const int jfirst = c0 - 31;
      const int pieces = kend * NP / 2;
      for (int e = lane; e < pieces; e += 32) {
        const int kk = e / (NP / 2);
        const int jj = jfirst + kk;
        if (jj >= 0 && jj < cols) {
          const double2 v = *reinterpret_cast<const double2*>(s_out + 2 * e);
          __stcg(reinterpret_cast<double2*>(colbuf + static_cast<size_t>(jj) * NP + (2 * e - kk * NP)), v);
        }
      }
      // columns handed up before / after this chunk
      const int done0 = min(max(c0 - 31, 0), cols);
      const int done1 = min(max(c0 + kend - 31, 0), cols);
      if (done1 > done0 && (done1 == cols || done1 / kPublish != done0 / kPublish)) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(prog_row + b, base + done1);
      }
    }
  }
  if (!has_above && P.bands > 1) {
    // the last band publishes completion too: the slot's next pair (p + slots)
    // may only rewrite the column buffer once this band has read all of it
    cp_async_wait<0>();
    __syncwarp();
    if (lane == 0) st_release_gpu(prog_row + b, base + cols);
  }
  if (jkey != ~0u) atomicMin(P.err + out, err_key(i, jkey >> 2, jkey & 3u));
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
    if (*reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0) return;
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
