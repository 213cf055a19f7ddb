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
#include <type_traits>

#include "sk_device.cuh"

namespace skb {

#ifndef SK_PUBLISH
#define SK_PUBLISH 16
#endif
// columns per progress publication (streaming schedule): one per chunk --
// single pairs, which the hand-over lag bounds, run 10 % faster than at 32
constexpr int kPublish = SK_PUBLISH;
#ifndef SK_SWEEP_WARPS
#define SK_SWEEP_WARPS 1
#endif
// Warps per CTA.  Warps are fully independent; one-warp CTAs avoid losing
// residency to CTA-granular register allocation.
constexpr int kSweepWarps = SK_SWEEP_WARPS;
// Resident one-warp CTAs per SM the register allocation must allow: each
// SM sub-partition holds 16K registers, so <= 168 registers/thread gives 3
// warps per sub-partition (12 per SM), more gives only 2.  Orders up to 10
// fit 168 without spills; larger orders keep the unconstrained allocation.
#ifndef SK_MIN_BLOCKS
#define SK_MIN_BLOCKS 0
#endif
__host__ __device__ constexpr int sweep_min_blocks(int N) {
  return SK_MIN_BLOCKS > 0 ? SK_MIN_BLOCKS : (N >= 1 && N <= 10 ? 12 : 1);
}

// Rows per lane: one tile row per lane, 32-row bands.  (Two rows per lane --
// 64-row bands, two independent tiles per step -- measured slower on B200:
// N = 8, d = 8, 256 x 4096^2: 77 vs 68 ms at 200 registers and 8 warps/SM.)
__host__ __device__ constexpr int rows_per_lane(int) { return 1; }
// columns per staging group / delta batch
#ifndef SK_CHUNK
#define SK_CHUNK 16
#endif
__host__ __device__ constexpr int chunk_cols(int) { return SK_CHUNK; }
// dx ring rows (power of two >= 32 + 2 chunks)
__host__ __device__ constexpr int ring_rows(int) { return 64; }

struct SweepParams {
  const double* xinc;             // increments of the column series (first series, x)
  const double* yinc;             // increments of the row series (second series, y)
  const uint32_t* pair_x;         // launch-local pair -> x series index
  const uint32_t* pair_y;         // launch-local pair -> y series index
  const uint32_t* pair_out;       // launch-local pair -> output slot
  unsigned long long sx, sy;      // elements between consecutive series
  const double* w65;              // N == 0: W table, row stride 65 (device memory)
  int dim, order;                 // dim: logical d
  int ld;                         // row stride of the increments (DP, or d rounded up to 4 when DP == 0)
  // DP == 0 table mode (the table fits the memory budget): rho (rows x cols,
  // row-major) per launch-local pair, formed by the DMMA GEMM beforehand;
  // null: the band CTAs' producer warps form rho in shared memory
  const double* rho_tab;
  unsigned long long tab_stride;  // elements per pair in rho_tab
  int rows, cols, bands, npairs, group, slots;
  unsigned flags;
  double* abuf;                   // slots x cols x NP
  unsigned long long* prog;       // slots x bands progress counters
  unsigned* queue;                // unit counter
  unsigned long long* watchdog;   // [0] abort flag, [1..4] first stuck wait (p, b, need, seen)
  unsigned long long watchdog_ns; // give up a dependency wait after this long
  int start_lag;                  // columns the band below must be ahead before a band starts
  // DP == 0 table mode, one pair per launch group, streaming: each CTA claims
  // rho_bands(N) consecutive bands per round, and a band whose neighbour
  // below is the previous warp of the same CTA takes its alpha from that
  // warp's shared-memory ring (CTA-scope counters) instead of the column
  // buffer in global memory (release to L2, poll, staging copy)
  int intra;
  // table mode beside a running GEMM (cfg 4 overlap): the GEMM counts the
  // 64 x 64 tiles written per 64-row block (rho_ready[pair * rho_ready_nrb +
  // block], rho_ready_need when complete) and a band starts once its block is
  // done.  slot_stride (doubles, > 0): the compact table-mode slot layout and
  // rho_bands(N) sweep warps per CTA (no producer warps), so GEMM CTAs fit
  // beside the sweep CTA.  Null / 0: the table is complete at launch.
  const unsigned* rho_ready;
  unsigned rho_ready_need;
  int rho_ready_nrb;
  int slot_stride;
  double dot_err;                 // EXACT, N > 0: bound on |fused dot - sequential dot| for any tile
  double* values;                 // per output slot: K(1,1)
  unsigned long long* err;        // per output slot: min error key (init ~0)
  unsigned long long* maxrho;     // per output slot: max |delta| bits (init 0) or null
  // Only the maximum over every pair of the launch is wanted (a Gram's
  // max_abs_increment_product without per-pair values): one shared running
  // max, so tiles below the launch's max so far skip the exact dot; the
  // per-slot values are then lower bounds only.  Null: per-pair maxima.
  unsigned long long* maxrho_all;
  double* grid;                   // per output slot: lx x ly knot grid, or null
  double* diag;                   // per output slot: K at tiles (i, i), or null
  unsigned long long grid_stride, diag_stride;
  // Long pair over several GPUs (block-cyclic strips):
  // the bands are cut into blocks of xblock bands dealt round-robin over
  // xgpus GPUs -- this launch sweeps the blocks k with k mod xgpus == xrank,
  // in increasing order (round r = k / xgpus), one column buffer per round.
  // With xexch set, every block boundary hands alpha over through exchange
  // buffers: block k's bottom band reads xin_abuf[r] / waits on xin_prog[r]
  // (this GPU's memory, written by the GPU of block k - 1), block k's top band
  // writes xout_abuf[r'] / publishes xout_prog[r'] (the next GPU's exchange
  // area, peer memory; r' = (k + 1) / xgpus), system-scope release/acquire.
  // One GPU, one launch: xgpus = 1, xblock = bands, xexch = 0.
  // xemul: ONE launch sweeps every band of all xgpus virtual GPUs (global band
  // order; the test of the multi-GPU indexing on one GPU): GPU g's round r
  // uses column buffer / exchange slot g * xrounds + r.
  int xgpus, xrank, xblock, xexch, xemul, xrounds;
  const double* xin_abuf;             // rounds x cols x NP
  const unsigned long long* xin_prog;  // rounds x kXProg
  double* xout_abuf;
  unsigned long long* xout_prog;
  // Segment-DAG mode (seg_cols > 0): the unit is (pair, band, segment), a
  // run of seg_cols steps of one band.  Band b's segment s covers steps
  // [s L - b H, (s+1) L - b H) (L = seg_cols, H = rows per band), so the
  // band below has produced every alpha a segment reads once its own segment
  // s is done: a unit runs only when both inputs -- (b, s-1) and (b-1, s) --
  // are complete and never waits inside.  Units become ready through
  // dependency counters (dep, per slot x band x segment) and a ready ring
  // (rq); bands carry their lane state between segments in susp records.
  int seg_cols, segs_per_band;
  unsigned units_total;
  int units_pair_streaming;  // bands per pair in this launch (streaming schedule)
  double* susp;
  unsigned* dep;
  unsigned* rq;   // ready list, units_total cells
  unsigned* ctr;  // one 128-byte line each: [0] ready head, [kCtrLine] tail
};

constexpr int kCtrLine = 32;  // u32 words per counter line
constexpr int kXProg = 16;    // u64 words between exchange progress counters (128 B)

// sweep_band outcomes
constexpr int kBandDone = 0, kBandAbort = 2;

__host__ __device__ constexpr int susp_record_doubles(int N) {
  return 32 * rows_per_lane(N) * (((N > 0 ? N + 1 : kMaxOrder + 1) + 1) & ~1) * 2;
}

// segment geometry of band b (rows per band H = 32 R)
struct SegRange {
  int lo, hi;  // first / last segment index of the band
};
__host__ __device__ inline int band_steps(int rows, int cols, int b, int H) {
  return cols + min(H, rows - b * H) - 1;
}
__host__ __device__ inline SegRange seg_range(int rows, int cols, int b, int H, int L) {
  return {b * H / L, (band_steps(rows, cols, b, H) - 1 + b * H) / L};
}

constexpr unsigned kFlagStrictCorner = 1u;
constexpr unsigned kFlagWFault = 4u;
// Internal: form and check every tile's total.  Without it (throughput
// launches) a band forms totals only in the chunks that can hold its pair's
// final tile; a non-finite total anywhere else still reaches the final value
// (non-finite series propagate through every later tile to the corner), and
// the host sweeps any pair that ends non-finite or flagged again with this
// bit set, which reports the reference's first failing tile exactly.
constexpr unsigned kFlagAllTotals = 1u << 8;
// Internal: run the literal (bit-identical) kernel whatever the order -- the
// strict-corner re-sweep of pairs the register kernels screened.
constexpr unsigned kFlagLiteral = 1u << 9;

__host__ __device__ constexpr int series_len(int N) { return N > 0 ? N + 1 : kMaxOrder + 1; }
__host__ __device__ constexpr int col_stride(int N) { return (series_len(N) + 1) & ~1; }
// dx ring row stride in doubles: 16-byte rows padded so that the 8 lanes of
// an LDS.128 phase (columns j, j-1, ..., j-7) hit distinct bank groups.
__host__ __device__ constexpr int ring_stride(int DP) { return DP <= 2 ? 2 : DP + 2; }
// per warp: band-below alpha stage (2 groups) | lane-to-lane alpha slots
// (32 R) | lane 31's top-row outputs of the chunk | dx ring (DP > 0) | delta
// stage (R x chunk x 32; x2 for the asynchronously staged table, DP = 0)
// d = 9..16 (DP = 16): the top lane stores its alpha' straight to global
// memory instead of parking a chunk of them in shared memory, which keeps the
// per-warp stage under 1/12 of the SM's shared memory (12 warps resident)
// Measured (cfg-5 shape, d = 16): parking the top lane's alpha' in shared
// memory and handing it up per chunk beats per-step global stores (550 vs 560
// ms per Gram of 64 members) once the delta stage is gone (inline deltas), so
// every register kernel parks.
#ifndef SK_DIRECT_OUT_MIN_DP
#define SK_DIRECT_OUT_MIN_DP 32
#endif
__host__ __device__ constexpr bool direct_top_out(int DP) { return DP >= SK_DIRECT_OUT_MIN_DP; }
// the chunk's deltas are staged in shared memory only where they are formed
// per chunk: the literal kernels (exact sequential dots); the register
// kernels form each tile's product inside the step (d <= 16)
__host__ __device__ constexpr bool chunk_deltas(int N, int DP, bool lit) { return DP > 0 && (N == 0 || lit); }
// lane-to-lane alpha slot buffers: two (written at step s into buffer s mod 2,
// read at step s + 1), so one warp barrier per step orders both the reads
// before the rewrite and the writes before the reads
#ifndef SK_PASS_BUFS
#define SK_PASS_BUFS 2
#endif
constexpr int kPassBufs = SK_PASS_BUFS;
__host__ __device__ constexpr int stage_doubles_per_warp(int N, int DP, bool lit = false) {
  return 2 * chunk_cols(rows_per_lane(N)) * col_stride(N) + kPassBufs * 32 * rows_per_lane(N) * col_stride(N) +
         (direct_top_out(DP) ? 0 : chunk_cols(rows_per_lane(N)) * col_stride(N)) +
         (DP > 0 ? ring_rows(rows_per_lane(N)) * ring_stride(DP) : 0) +
         (chunk_deltas(N, DP, lit) ? rows_per_lane(N) * chunk_cols(rows_per_lane(N)) * 32 : 0);
}

// ---- large d (DP == 0): the increment products are produced INSIDE the
// sweep's CTA, never materialised in HBM.  Each band has a sweep warp (the
// consumer) and a producer warp that computes the band's rho block by block
// -- 32 rows x kRhoB columns, contracted over d with FP64 tensor-core MMA
// (mma.sync m8n8k4, SASS DMMA), or with the reference's sequential non-FMA
// dot for the literal kernel -- into a shared-memory ring of kRhoRB blocks
// that the sweep warp reads at step s, lane t, column s - t.  Flow control:
// two counters in shared memory (blocks produced, chunks consumed) with
// CTA-scope release/acquire.  Memory per pair stays O(l (N+d)) whatever d
// is (wavefront.cpp:100-105,146-149 form rho per tile too).
#ifndef SK_RHO_KC
#define SK_RHO_KC 16
#endif
#ifndef SK_RHO_STAGES
#define SK_RHO_STAGES 3
#endif
constexpr int kRhoB = 32;                 // columns per produced block (4 MMA n-tiles)
#ifndef SK_RHO_RB
#define SK_RHO_RB 2
#endif
constexpr int kRhoRB = SK_RHO_RB;         // ring blocks
constexpr int kRhoW = kRhoB * kRhoRB;     // ring columns (power of two)
constexpr int kRhoKC = SK_RHO_KC;         // k (coordinate) chunk staged per cp.async group
constexpr int kRhoKS = kRhoKC + 4;        // staging row stride: conflict-free fragment loads
constexpr int kRhoStages = SK_RHO_STAGES; // cp.async pipeline depth
static_assert((kRhoW & (kRhoW - 1)) == 0, "ring width must be a power of two");
static_assert(kRhoW * 32 >= 2 * SK_CHUNK * 32, "table mode stages two chunks of deltas in the ring's memory");

__host__ __device__ constexpr int rho_ring_doubles() { return kRhoW * 32; }
__host__ __device__ constexpr int rho_stage_doubles() { return kRhoStages * (32 + kRhoB) * kRhoKS; }
// DP == 0: one band's shared memory -- sweep stage | rho ring | producer staging
__host__ __device__ constexpr int rho_slot_doubles(int N) {
  return stage_doubles_per_warp(N, 0) + rho_ring_doubles() + rho_stage_doubles();
}
// A DP == 0 CTA sweeps rho_bands(N) bands (one CTA per SM): warps
// 0..bands-1 are their sweep warps, the next `bands` warps their producers.
// At most one sweep warp per SM sub-partition: warp w of a CTA runs on
// sub-partition w mod 4, and two latency-bound sweep warps sharing one ran
// ~2x slower (measured on cfg 4's sweep: one-warp band CTAs 19.3 ms vs
// two-warp CTAs -- sweep warps on sub-partitions 0, 2, 0 -- 36.5 ms).  Four
// bands when their shared memory fits the SM (N <= 13), fewer otherwise.
constexpr int kSmemDoubles = 232448 / 8;  // 227 KB per CTA
#ifndef SK_RHO_MAXBANDS
#define SK_RHO_MAXBANDS 4
#endif
__host__ __device__ constexpr int rho_bands(int N) {
  return kSmemDoubles / rho_slot_doubles(N) >= SK_RHO_MAXBANDS ? SK_RHO_MAXBANDS : kSmemDoubles / rho_slot_doubles(N);
}
__host__ __device__ constexpr int sweep_warps(int N, int DP) { return DP == 0 ? 2 * rho_bands(N) : kSweepWarps; }
// bands swept concurrently by one CTA
__host__ __device__ constexpr int band_workers(int N, int DP) { return DP == 0 ? rho_bands(N) : kSweepWarps; }
// dynamic shared memory of one CTA (doubles)
__host__ __device__ constexpr int sweep_smem_doubles(int N, int DP, bool lit = false) {
  return DP > 0 ? kSweepWarps * stage_doubles_per_warp(N, DP, lit) : rho_bands(N) * rho_slot_doubles(N);
}

// producer / consumer hand-shake of a DP == 0 band CTA (static shared memory)
struct RhoCtl {
  unsigned p, b;        // the unit: pair (launch-local) and band
  int c_begin, c_end;   // its chunk range
  unsigned stop;        // no more units: producers exit
  unsigned abort;       // the consumer abandoned the unit (watchdog)
  unsigned prod;        // blocks < prod are in the ring (absolute block index)
  unsigned cons;        // chunks < cons are done (absolute chunk index)
  unsigned up_prod;     // intra: steps whose top-row alpha' is in this band's ring
  unsigned up_cons;     // intra: steps of this band's ring the band above has copied
};
// intra hand-over ring: the top row's alpha' of the last kUpChunks chunks
constexpr int kUpChunks = 4;
// shared memory a compact table-mode sweep CTA requests: > half the SM's
// 228 KB, so two never share an SM, and leaves room for two 41 KB GEMM CTAs
#ifndef SK_TABLE_CTA_KB
#define SK_TABLE_CTA_KB 118
#endif
constexpr size_t kTableCtaSmem = SK_TABLE_CTA_KB * 1024;
// compact table-mode slot (SweepParams::slot_stride): stage | staged table
// deltas (2 x K x 32) | intra ring
__host__ __device__ constexpr int table_slot_doubles(int N) {
  return stage_doubles_per_warp(N, 0) + 2 * chunk_cols(rows_per_lane(N)) * 32 +
         kUpChunks * chunk_cols(rows_per_lane(N)) * col_stride(N);
}
constexpr unsigned kIntraBar = 15;  // named barrier of the CTA's sweep warps (intra rounds)

__device__ __forceinline__ unsigned ld_acquire_cta_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "r"(v) : "memory");
}
__device__ __forceinline__ void named_bar_sync(unsigned id, unsigned threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
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
#ifdef SK_PROFILE_WAITS
// per-unit trace (diagnostic build only): {p | b << 20 | smid << 40, start ns, end ns, wait ns}
constexpr unsigned kTraceUnits = 1u << 16;
__device__ unsigned long long g_utrace[kTraceUnits * 4];
__device__ unsigned long long g_wwait[1u << 14];
__device__ unsigned g_tidx;
#endif

#ifndef SK_POLL_CAP
#define SK_POLL_CAP 256  // ns: longest back-off between two polls of a progress counter
#endif
static __device__ __noinline__ bool wait_progress_slow(const unsigned long long* ptr, unsigned long long need,
                                                       unsigned long long& seen, unsigned long long* wd,
                                                       unsigned long long limit_ns, unsigned p, unsigned b,
                                                       bool sys) {
  // poll with relaxed loads (no L1 invalidation per poll) and a growing
  // back-off; the acquire is taken once the value is there
  const unsigned long long t0 = globaltimer_ns();
  unsigned ns = 32;
  for (unsigned it = 1;; ++it) {
    __nanosleep(ns);
    if (ns < SK_POLL_CAP) ns += ns >> 1;
    if ((sys ? ld_relaxed_sys(ptr) : ld_relaxed_gpu(ptr)) >= need) break;
    if ((it & 15) == 0) {
      if (*reinterpret_cast<volatile unsigned long long*>(wd) != 0) return false;
      if (globaltimer_ns() - t0 > limit_ns) {
        if ((threadIdx.x & 31) == 0 && atomicCAS(wd, 0ull, 1ull) == 0ull) {
          wd[1] = p;
          wd[2] = b;
          wd[3] = need;
          wd[4] = sys ? ld_relaxed_sys(ptr) : ld_relaxed_gpu(ptr);
        }
        return false;
      }
    }
  }
  seen = sys ? ld_acquire_sys(ptr) : ld_acquire_gpu(ptr);
  return true;
}

__device__ __forceinline__ bool wait_progress(const SweepParams& P, const unsigned long long* ptr,
                                              unsigned long long need, unsigned long long& seen, unsigned p,
                                              unsigned b, bool sys = false) {
  if (seen >= need) return true;
  const unsigned long long v = sys ? ld_acquire_sys(ptr) : ld_acquire_gpu(ptr);  // every lane polls one word
  if (v >= need) {
    seen = v;
    return true;
  }
#ifdef SK_PROFILE_WAITS
  const long long t0 = clock64();
  const unsigned long long g0 = globaltimer_ns();
  const bool ok = wait_progress_slow(ptr, need, seen, P.watchdog, P.watchdog_ns, p, b, sys);
  if ((threadIdx.x & 31) == 0) {
    g_wwait[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] += globaltimer_ns() - g0;
    atomicAdd(reinterpret_cast<unsigned long long*>(P.watchdog + 6), clock64() - t0);
    // [5]: cycles of waits whose target is the band's first chunks (start-up lag)
    if (need - static_cast<unsigned long long>(p) * (P.cols + 1) <= max(64, P.start_lag))
      atomicAdd(reinterpret_cast<unsigned long long*>(P.watchdog + 5), clock64() - t0);
  }
  return ok;
#else
  return wait_progress_slow(ptr, need, seen, P.watchdog, P.watchdog_ns, p, b, sys);
#endif
}

// one look at a progress counter, no waiting; warp-uniform: true only when
// every lane's own acquire saw the count (each lane then reads what it covers)
__device__ __forceinline__ bool poll_progress(const unsigned long long* ptr, unsigned long long need,
                                              unsigned long long& seen, bool sys = false) {
  bool ok = seen >= need;
  if (!__all_sync(0xffffffffu, ok)) {
    const unsigned long long v = sys ? ld_acquire_sys(ptr) : ld_acquire_gpu(ptr);
    if (v >= need) seen = v;
    ok = __all_sync(0xffffffffu, v >= need);
  }
  return ok;
}

// ---- ready list (segment-DAG mode, lane 0 only) ------------------------------
// Every unit is pushed exactly once (the initial ones by the host), so the
// list has units_total cells and never wraps: push takes the next cell with
// the tail counter and publishes the unit (+1) with a release store; pop
// takes the next cell with the head counter (always succeeds) and waits for
// its unit.  A warp whose cell index is past the end has nothing left to do.
__device__ __forceinline__ void rq_push(const SweepParams& P, unsigned unit) {
  const unsigned t = atomicAdd(P.ctr + kCtrLine, 1u);
  st_release_u32(P.rq + t, unit + 1u);
}
// one input of unit (slot-local index `di`, launch unit id `unit`) is
// complete; the last of its `ndep` inputs queues it.  acq_rel: the unit's
// runner sees every predecessor's stores.
__device__ __forceinline__ void dep_arrive(const SweepParams& P, size_t di, unsigned ndep, unsigned unit) {
  if (atom_add_acq_rel_u32(P.dep + di, 1u) + 1u == ndep) rq_push(P, unit);
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
// Steps [c_begin K, min(c_end K, steps)) of band b of pair p.  Streaming
// mode (P.seg_cols == 0): the whole band (c_begin = 0, c_end = INT_MAX),
// waiting on the band below's progress counter.  Segment mode: one segment,
// all inputs complete; `restore` loads the band's lane state from its record
// (not the band's first segment), `save` stores it (not the last).
template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
__device__ __forceinline__ int sweep_band(const SweepParams& P, unsigned p, unsigned b, int lane,
                                          double* __restrict__ smem, int c_begin, int c_end, bool restore,
                                          bool save, RhoCtl* ctl) {
  constexpr int R = rows_per_lane(N);
  constexpr int K = chunk_cols(R);
  constexpr int RING = ring_rows(R);
  constexpr int NA = series_len(N);
  constexpr int NP = col_stride(N);
  constexpr int XS = ring_stride(DP);
  constexpr int kStage = K * NP;
#ifndef SK_INLINE_DELTA
#define SK_INLINE_DELTA 1
#endif
  // increments products formed inside the step (not per chunk) where the
  // registers allow it: d <= 8, register kernels, no exact max.  Measured:
  // 256 x 4096^2 62.95 vs 63.5 ms; at d = 16 it spills and gains nothing.
  // Register kernels form each tile's increment product inside the step (its
  // loads and FMAs overlap the tile math's dependency chains); the EXACT
  // variant tracks the lane's largest fast |delta| per chunk and re-forms the
  // chunk's products with the sequential dot only when that could raise the
  // exact max (chunk end).  Measured: 256 x 4096^2 at d = 16, 64.7 vs 69.9 ms
  // against per-chunk products in shared memory.
  constexpr bool kInlineDelta = SK_INLINE_DELTA && DP > 0 && N > 0 && !LIT && R == 1;
  static_assert(kInlineDelta == (DP > 0 && !chunk_deltas(N, DP, LIT)) || !SK_INLINE_DELTA,
                "shared-memory delta stage exactly where deltas are formed per chunk");
  // LIT: the literal (bit-identical) arithmetic at a compile-time order N,
  // unscaled series in registers (strict-corner re-sweeps); like N == 0 it
  // needs the exact deltas and every total
  static_assert(!LIT || (N > 0 && EXACT && EXTRAS), "LIT variants are <N > 0, EXACT, EXTRAS>");
  constexpr bool kLiteral = N == 0 || LIT;
  double* s_alpha = smem;                                   // 2 x K x NP
  double* s_pass = s_alpha + 2 * kStage;                    // 32 R x NP: slot (32 r + t) = row 32 r + t
  double* s_out = s_pass + kPassBufs * 32 * R * NP;         // K x NP
  constexpr int kPassBuf = 32 * R * NP;  // one slot buffer
  // the slot buffer step s reads (written at step s - 1) / writes
  auto pass_in = [&](int s) { return s_pass + (kPassBufs == 2 ? ((s - 1) & 1) * kPassBuf : 0); };
  auto pass_out = [&](int s) { return s_pass + (kPassBufs == 2 ? (s & 1) * kPassBuf : 0); };
  double* s_ring = s_out + (direct_top_out(DP) ? 0 : kStage);  // RING x XS (DP > 0)
  double* s_delta = s_ring + (DP > 0 ? RING * XS : 0);      // [r][k][lane] (DP > 0)
  // DP == 0: the producers' rho ring, column c of row t at [(c mod kRhoW) * 32 + t];
  // table mode: the same memory holds the staged table deltas [buf][k][lane]
  const double* rho_ring = smem + stage_doubles_per_warp(N, 0);
  const bool tab_mode = DP == 0 && P.rho_tab != nullptr;
  double* s_tab = smem + stage_doubles_per_warp(N, 0);
  const double* tab = DP > 0 || !tab_mode ? nullptr : P.rho_tab + static_cast<size_t>(p) * P.tab_stride;
  // intra-CTA hand-over (SweepParams::intra): this band's ring after the
  // staged table deltas; the band below is the previous warp's slot
  constexpr int kUpRing = kUpChunks * K;  // steps held (power of two)
  static_assert((kUpRing & (kUpRing - 1)) == 0, "intra ring index by mask");
  double* const up_ring = smem + stage_doubles_per_warp(N, 0) + 2 * K * 32;
  static_assert(DP > 0 || N == 0 || 2 * K * 32 + kUpRing * NP <= rho_ring_doubles() + rho_stage_doubles(),
                "intra ring fits the slot's producer memory (unused in table mode)");
  const int n = N > 0 ? N + 1 : P.order + 1;
  const int rows = P.rows, cols = P.cols;
  const int row0 = static_cast<int>(b) * 32 * R;
  const int rb = min(32 * R, rows - row0);
  // strips: one column buffer per block round; pairs: slot of the pair
  const unsigned blk = b / static_cast<unsigned>(P.xblock);
  const unsigned G = static_cast<unsigned>(P.xgpus);
  // slot of block k's round on its GPU (xemul: per virtual GPU)
  auto round_slot = [&](unsigned k) { return P.xemul ? (k % G) * static_cast<unsigned>(P.xrounds) + k / G : k / G; };
  const unsigned slot = P.xgpus > 1 || P.xexch ? round_slot(blk) : p % static_cast<unsigned>(P.slots);
  const unsigned long long base = static_cast<unsigned long long>(p) * static_cast<unsigned long long>(cols + 1);
  double* colbuf = P.abuf + static_cast<size_t>(slot) * static_cast<size_t>(cols) * NP;
  unsigned long long* prog_row = P.prog + static_cast<size_t>(slot) * P.bands;
  const bool has_below = b > 0;
  const bool has_above = b + 1 < static_cast<unsigned>(P.bands);
  // (the kernel's slot of this warp: warp mod rho_bands)
  const int kslot = DP == 0 ? static_cast<int>(threadIdx.x >> 5) % rho_bands(N) : 0;
  const bool intra_in = DP == 0 && N > 0 && P.intra && has_below && kslot > 0;
  const bool intra_out = DP == 0 && N > 0 && P.intra && has_above && kslot + 1 < rho_bands(N);
  RhoCtl* const below_ctl = ctl - (intra_in ? 1 : 0);
  const double* const below_ring =
      up_ring - (intra_in ? (P.slot_stride > 0 ? P.slot_stride : rho_slot_doubles(N)) : 0);  // the kernel's slot stride
  // a dependency on the band below through global memory
  const bool gdep = P.seg_cols == 0 && has_below && !intra_in;
  // intra hand-over wait on a CTA-scope counter (lane 0 polls, the warp
  // follows; gives up when the launch aborts or after the watchdog time)
  auto intra_wait = [&](const unsigned* ctr, unsigned need) -> bool {
    int stuck = 0;
    if (lane == 0 && ld_acquire_cta_u32(ctr) < need) {
      const unsigned long long t0 = globaltimer_ns();
      unsigned ns = 16;
      while (ld_acquire_cta_u32(ctr) < need) {
        __nanosleep(ns);
        if (ns < 128) ns *= 2;
        if (*reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0) {
          stuck = 1;
          break;
        }
        if (globaltimer_ns() - t0 > P.watchdog_ns) {
          if (atomicCAS(P.watchdog, 0ull, 1ull) == 0ull) {
            P.watchdog[1] = p;
            P.watchdog[2] = b;
            P.watchdog[3] = need;
            P.watchdog[4] = *reinterpret_cast<const volatile unsigned*>(ctr);
          }
          stuck = 1;
          break;
        }
      }
    }
    const bool ok = __shfl_sync(0xffffffffu, stuck, 0) == 0;
    __syncwarp();  // lane 0's acquire before every lane reads what it covers
    return ok;
  };
  // table beside a running GEMM: this band's 64-row block of the table
  auto rows_ready = [&]() -> bool {
    const unsigned* ctr = P.rho_ready + static_cast<size_t>(p) * P.rho_ready_nrb + row0 / 64;
    const unsigned need = P.rho_ready_need;
    int stuck = 0;
    if (lane == 0 && ld_acquire_u32(ctr) < need) {
      const unsigned long long t0 = globaltimer_ns();
      unsigned ns = 64;
      while (ld_acquire_u32(ctr) < need) {
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
        if (*reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0 ||
            globaltimer_ns() - t0 > P.watchdog_ns) {
          if (atomicCAS(P.watchdog, 0ull, 1ull) == 0ull) {
            P.watchdog[1] = p;
            P.watchdog[2] = b;
            P.watchdog[3] = need;
            P.watchdog[4] = *reinterpret_cast<const volatile unsigned*>(ctr);
          }
          stuck = 1;
          break;
        }
      }
    }
    const bool ok = __shfl_sync(0xffffffffu, stuck, 0) == 0;
    __syncwarp();  // lane 0's acquire before every lane gathers table rows
    return ok;
  };
  // where this band's alpha comes from / goes to: the pair's column buffer,
  // or a cross-strip exchange buffer (multi-GPU long pair)
  const bool xin = P.xexch && has_below && b % static_cast<unsigned>(P.xblock) == 0;
  const bool xout = P.xexch && has_above && (b + 1) % static_cast<unsigned>(P.xblock) == 0;
  const size_t xstride = static_cast<size_t>(cols) * NP;
  const unsigned rin = round_slot(blk);
  const unsigned rout = round_slot(blk + 1);
  const double* in_buf = xin ? P.xin_abuf + rin * xstride : colbuf;
  const unsigned long long* in_prog = xin ? P.xin_prog + rin * kXProg : prog_row + (has_below ? b - 1 : 0);
  double* out_buf = xout ? P.xout_abuf + rout * xstride : colbuf;
  unsigned long long* out_prog = xout ? P.xout_prog + rout * kXProg : prog_row + b;
  const unsigned out = P.pair_out[p];
  const bool strict = (P.flags & kFlagStrictCorner) != 0;
  const bool fault = (P.flags & kFlagWFault) != 0;
  // every tile's total: literal kernels, the re-sweep flag, knot grids; the
  // knot diagonal needs them only in the chunks holding a tile (i, i)
  const bool all_totals = kLiteral || (P.flags & kFlagAllTotals) != 0 || (EXTRAS && P.grid != nullptr);
  const bool band_top = row0 + 32 * R >= rows;  // the band holds the pair's last row
  const bool streaming = P.seg_cols == 0;
  double* const rec = streaming ? nullptr
                                : P.susp + (static_cast<size_t>(slot) * P.bands + b) *
                                               static_cast<size_t>(susp_record_doubles(N));

  // Slot hand-over: band 0 of pair p rewrites the column buffer that the last
  // band of the slot's previous pair (p - slots) reads.  (Segment mode: the
  // pair's first unit is queued only once the previous pair has finished.)
  if (streaming && b == 0 && has_above && p >= static_cast<unsigned>(P.slots)) {
    unsigned long long seen0 = 0;
    if (!wait_progress(P, prog_row + (P.bands - 1), static_cast<unsigned long long>(p - P.slots) * (cols + 1) + cols,
                       seen0, p, b))
      return kBandAbort;
  }

  // per tile r of this lane: row i_r = row0 + 32 r + lane, column s - lane - 32 r
  int irow[R];
  bool row_ok[R], last_row[R];
  const double* yrow[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    irow[r] = row0 + 32 * r + lane;
    row_ok[r] = 32 * r + lane < rb;
    last_row[r] = row_ok[r] && irow[r] == rows - 1;
    // increments are stored with row stride DP behind one leading zero row
    yrow[r] = DP > 0 ? P.yinc + P.pair_y[p] * P.sy + static_cast<size_t>(row_ok[r] ? irow[r] + 1 : 0) * DP : nullptr;
  }
  const double* xser = DP > 0 ? P.xinc + P.pair_x[p] * P.sx + DP : nullptr;  // row j at xser + j * DP
  // DP == 0: this pair's increments (exact dots of the EXACT candidates)
  const double* xrows0 = DP > 0 ? nullptr : P.xinc + P.pair_x[p] * P.sx + P.ld;  // row j at xrows0 + j * ld
  const double* yrows0 = DP > 0 ? nullptr : P.yinc + P.pair_y[p] * P.sy + P.ld;

  // Loop-carried register state: each tile's beta (the left edge of its next
  // tile), ping-ponged between A and B.  Before a tile's first column it runs
  // the delta = 0 tile on unit series, whose output is the unit series again,
  // so beta is e0 exactly at its first column without a select.
  double roA[R][NA], roB[R][NA];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int m = 0; m < NA; ++m) roA[r][m] = (m == 0) ? 1.0 : 0.0;
  // running exact max|delta| of this band: start from the pair's value so far
  // (a valid lower bound) so fewer tiles need the exact dot
  double mx = 0.0;
  // EXACT, inline products: the lane's largest fast |delta| in the chunk (bits)
  unsigned long long fmxb[R];
  const unsigned long long kLimitBits = static_cast<unsigned long long>(__double_as_longlong(kDeltaOverflowLimit));
#pragma unroll
  for (int r = 0; r < R; ++r) fmxb[r] = 0ull;
  if constexpr (EXACT && !kLiteral) {
    if (P.maxrho) mx = __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(P.maxrho + out)));
    if (P.maxrho_all)
      mx = fmax(mx, __longlong_as_double(static_cast<long long>(*reinterpret_cast<volatile unsigned long long*>(P.maxrho_all))));
  }
  unsigned jkey[R];  // (first failing column << 2) | code, per tile
#pragma unroll
  for (int r = 0; r < R; ++r) jkey[r] = ~0u;
  // the rows' increments stay in registers for the whole band: a reload per
  // chunk would miss L1, which every acquire of the progress counter invalidates
  double dyr[R][DP > 0 ? DP : 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if constexpr (DP > 0) {
#pragma unroll
      for (int c = 0; c < DP; c += 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(yrow[r] + c));
        dyr[r][c] = v.x;
        dyr[r][c + 1] = v.y;
      }
    } else {
      dyr[r][0] = 0.0;
    }
  }
  unsigned long long seen = 0;
  const int steps = cols + rb - 1;

  // ---- staging: group g = steps/columns [g K, g K + K): band-below alpha
  // (2 buffers) and dx (ring row = column mod RING; DP > 0) or the table
  // deltas of those steps (DP == 0 table mode, 2 buffers); one cp.async group
  // per g.
  auto stage_group = [&](int g) {
    const int col0 = g * K;
    const int ncol = max(0, min(K, cols - col0));
    if (has_below && !intra_in) {
      const double* src = in_buf + static_cast<size_t>(col0) * NP;
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
        cp_async_16(s_ring + (col & (RING - 1)) * XS + 2 * part, xser + static_cast<size_t>(col) * DP + 2 * part);
      }
    } else if (tab_mode) {
      // row-major table: lane t gathers rho(i, g K + k - t), zero-filled
      // outside the pair (8-byte cp.async, consecutive lanes -> consecutive
      // shared words)
      double* dst = s_tab + (g & 1) * K * 32 + lane;
      const double* trow = tab + static_cast<size_t>(row_ok[0] ? irow[0] : 0) * cols;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const int j = col0 + k - lane;
        const bool ok = row_ok[0] && j >= 0 && j < cols;
        cp_async_8_zfill(dst + k * 32, trow + (ok ? j : 0), ok);
      }
    }
    cp_async_commit();
  };
  if (!has_below) {
    // band 0: the bottom edge of the domain is the unit series in every column
    for (int e = lane; e < 2 * kStage; e += 32) s_alpha[e] = (e % NP == 0) ? 1.0 : 0.0;
  }
  if (restore) {
    // lane state at the segment boundary: beta (registers) and the
    // lane-to-lane alpha slots
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < NA; ++m)
        if (NA <= kMaxRegOrder + 1 || m < n) roA[r][m] = rec[(r * NP + m) * 32 + lane];
    double* const sp0 = pass_in(c_begin * K);
    for (int e = lane; e < 32 * R * NP; e += 32) sp0[e] = rec[32 * R * NP + e];
  } else {
    double* const sp0 = pass_in(c_begin * K);
    for (int e = lane; e < 32 * R * NP; e += 32) sp0[e] = (e % NP == 0) ? 1.0 : 0.0;
  }
  if constexpr (DP > 0) {
    // dx of the columns the lanes still need behind the first staged group,
    // [c K - 32 R, c K): zero below column 0 (zero increments => delta = 0,
    // which keeps a tile's beta at the unit series before its first column)
    const int h0 = c_begin * K - 32 * R;
    for (int e = lane; e < 32 * R * (DP / 2); e += 32) {
      const int c = e / (DP / 2), part = e - c * (DP / 2);
      const int col = h0 + c;
      double* dst = s_ring + (col & (RING - 1)) * XS + 2 * part;
      if (col < 0) {
        dst[0] = 0.0;
        dst[1] = 0.0;
      } else if (col < cols) {
        cp_async_16(dst, xser + static_cast<size_t>(col) * DP + 2 * part);
      }
    }
  }
  __syncwarp();
  // start no closer than start_lag columns behind the band below: bands of
  // one pair then run evenly spread in time instead of bunched at the
  // minimum hand-over distance, where every timing jitter becomes a wait
  if (gdep && !wait_progress(P, in_prog, base + min(cols, max(K, P.start_lag)), seen, p, b, xin))
    return kBandAbort;
  if (DP == 0 && tab_mode && P.rho_ready != nullptr && !rows_ready()) return kBandAbort;
  stage_group(c_begin);

  // one step = R tiles of this lane (one basic block, conditional work predicated)
  auto step = [&](bool TOT, int s, int k, const double* stage, const double* dl, double (&r_in)[R][NA],
                  double (&ro_out)[R][NA]) {
    double q[R][NA];
    // alpha: lane 0's first tile from the band below (stage); every other
    // tile from the slot of the row below -- slot index (32 r + t) - 1, so
    // lane 0's tile r >= 1 reads lane 31's tile r - 1
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double* src = (r == 0 && lane == 0) ? stage + k * NP : pass_in(s) + (32 * r + lane - 1) * NP;
      lds_series<NA>(src, q[r], n);
    }
    if constexpr (kPassBufs == 1) __syncwarp();  // every slot has been read before any is rewritten
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int j = s - lane - 32 * r;
      double delta;
      if constexpr (kInlineDelta) {
        // this tile's increment product, formed in the step (its loads and
        // FMAs overlap the tile math's dependency chains) with its guard
        const double* xr = s_ring + ((s - lane - 32 * r) & (RING - 1)) * XS;
        double e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int c = 0; c < DP; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(xr + c);
          e0 = fma(v.x, dyr[r][c], e0);
          e1 = fma(v.y, dyr[r][c + 1], e1);
        }
        delta = e0 + e1;
        const bool act = row_ok[r] && j >= 0 && j < cols;
        if constexpr (EXACT && DP >= 16) {
          // the guard and the running max on the bits of |delta| (integer
          // pipe; non-negative doubles order as their bit patterns, a NaN
          // above every finite value): !(|delta| <= limit) == bits > limit
          // bits.  Measured: Gram (d = 16, exact max) -0.65 %; slower for
          // d = 8 and without the exact max, which keep the FP64 compare.
          const unsigned long long dbits =
              static_cast<unsigned long long>(__double_as_longlong(delta)) & 0x7fffffffffffffffull;
          jkey[r] = min(jkey[r], (act && dbits > kLimitBits) ? (static_cast<unsigned>(j) << 2) | kErrDelta : ~0u);
          fmxb[r] = max(fmxb[r], act ? dbits : 0ull);
        } else {
          jkey[r] = min(jkey[r], (act && !(fabs(delta) <= kDeltaOverflowLimit))
                                     ? (static_cast<unsigned>(j) << 2) | kErrDelta
                                     : ~0u);
          if constexpr (EXACT)
            fmxb[r] = static_cast<unsigned long long>(__double_as_longlong(
                fmax(__longlong_as_double(static_cast<long long>(fmxb[r])), act ? fabs(delta) : 0.0)));
        }
      } else if constexpr (DP > 0) {
        delta = dl[(r * K + k) * 32 + lane];
      } else {
        delta = tab_mode ? dl[k * 32 + lane] : rho_ring[((s - lane) & (kRhoW - 1)) * 32 + lane];
      }
      double qo[NA];
      double total = 0.0;
      if constexpr (LIT) {
        total = tile_step_literal_reg<N>(q[r], r_in[r], delta, qo, ro_out[r], fault);
      } else if constexpr (N > 0) {
        // the total (non-finite check, wavefront.cpp:169-173; the final
        // value) only in TOT chunks -- see kFlagAllTotals
        tile_update_scaled<N>(q[r], r_in[r], delta, qo, ro_out[r], fault);
        if (TOT) total = scaled_total<N>(qo);
      } else {
        total = tile_step_literal(P.order, q[r], r_in[r], delta, P.w65, qo, ro_out[r]);
      }
      // alpha' up: the band's top row (lane 31, last tile) parks it for the
      // band above, every other row in its slot
      if constexpr (direct_top_out(DP)) {
        // every row in its slot (the top lane's slot is never read); the top
        // row's alpha' straight to the column buffer of the band above
        sts_series<NA>(pass_out(s) + (32 * r + lane) * NP, qo, n);
        if (r == R - 1) {
          const bool up = has_above && lane == 31 && j >= 0 && j < cols;
          double* dst = out_buf + static_cast<size_t>(up ? j : 0) * NP;
#pragma unroll
          for (int m = 0; m < NA; m += 2) st_global_cg2_if(up, dst + m, qo[m], m + 1 < NA ? qo[m + 1] : 0.0);
        }
      } else {
        sts_series<NA>((r == R - 1 && lane == 31) ? s_out + k * NP : pass_out(s) + (32 * r + lane) * NP, qo, n);
      }

      const bool active = row_ok[r] && j >= 0 && j < cols;
      // the reference's throw order inside a tile: delta guard (checked when
      // the chunk's deltas are formed), corner check, non-finite total
      // (wavefront.cpp:150-173); the first failing tile of the row wins
      const bool cm = strict & (kLiteral ? corner_mismatch(q[r][0], r_in[r][0], kCornerTol)
                                         : corner_screen(q[r][0], r_in[r][0]));
      const bool nf = (TOT || kLiteral) && !isfinite(total);
      const unsigned code = cm ? kErrCorner : (nf ? kErrNonFinite : 0u);
      const unsigned kk = (static_cast<unsigned>(j) << 2) | code;
      jkey[r] = min(jkey[r], (active && code != 0u) ? kk : ~0u);
      if (TOT || kLiteral) st_global_if(last_row[r] && j == cols - 1, P.values + out, total);
      if constexpr (EXTRAS) {
        if (P.grid)
          st_global_if(active,
                       P.grid + out * P.grid_stride + static_cast<size_t>(j + 1) * (rows + 1) + (irow[r] + 1),
                       total);
        if (P.diag) st_global_if(active && irow[r] == j, P.diag + out * P.diag_stride + irow[r], total);
      }
    }
    __syncwarp();  // slots written before the next step reads them
  };

  const int ngroups_in = (cols + K - 1) / K;
  const int ngroups = DP > 0 ? ngroups_in : (steps + K - 1) / K;
  // the chunk's increment products / table deltas (s_delta) with the delta guard
  auto form_deltas = [&](int c0, int kend, const double* dl) {
    // the chunk's increment products (tile r, step c0 + k -> column
    // c0 + k - t - 32 r) with the delta guard (wavefront.cpp:150-155) and max|delta|
#pragma unroll
    for (int r = 0; r < (kInlineDelta ? 0 : R); ++r) {
      const double (&dy)[DP > 0 ? DP : 1] = dyr[r];
#pragma unroll 1
      for (int k0 = 0; k0 < K; k0 += 4) {
        double dd[4];
        if constexpr (DP > 0) {
          // four columns at a time: all loads first, then four independent dots
          double dx[4][DP];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* xr = s_ring + ((c0 + k0 + u - lane - 32 * r) & (RING - 1)) * XS;
#pragma unroll
            for (int c = 0; c < DP; c += 2) {
              const double2 v = *reinterpret_cast<const double2*>(xr + c);
              dx[u][c] = v.x;
              dx[u][c + 1] = v.y;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if constexpr (EXACT && kLiteral) {
              dd[u] = exact_dot<DP>(dx[u], dy);  // the literal kernel repeats the reference bit for bit
            } else {
              double e0 = dx[u][0] * dy[0], e1 = dx[u][1] * dy[1];
#pragma unroll
              for (int c = 2; c < DP; c += 2) {
                e0 = fma(dx[u][c], dy[c], e0);
                e1 = fma(dx[u][c + 1], dy[c + 1], e1);
              }
              dd[u] = e0 + e1;
            }
            s_delta[(r * K + k0 + u) * 32 + lane] = dd[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            dd[u] = tab_mode ? dl[(k0 + u) * 32 + lane] : rho_ring[((c0 + k0 + u - lane) & (kRhoW - 1)) * 32 + lane];
        }
        unsigned cand = 0u;  // EXACT, N > 0: tiles whose exact |delta| could raise the running max
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + u;
          const int j = c0 + k - lane - 32 * r;
          const bool act = row_ok[r] && j >= 0 && j < cols && k < kend;
          const double ad = fabs(dd[u]);
          if constexpr (EXACT && kLiteral) mx = fmax(mx, act ? ad : 0.0);  // dd is exact here
          if constexpr (EXACT && !kLiteral) cand |= (act && ad + P.dot_err >= mx) ? 1u << u : 0u;
          const unsigned kk = (static_cast<unsigned>(j) << 2) | kErrDelta;
          jkey[r] = min(jkey[r], (act && !(ad <= kDeltaOverflowLimit)) ? kk : ~0u);
        }
        if constexpr (EXACT && !kLiteral) {
          // exact max|delta| (bit-identical to max_abs_rho) without an exact
          // dot per tile: |fast - sequential| <= dot_err, so only a tile whose
          // fast |delta| + dot_err reaches the running exact max can raise it
          // -- rare once the max has settled; those get the sequential dot,
          // re-reading their dx row from the ring (DP > 0) or both rows from
          // global memory (DP == 0)
          if (__any_sync(0xffffffffu, cand != 0u)) {
#pragma unroll 1
            for (int u = 0; u < 4; ++u)
              if ((cand >> u) & 1u) {
                if constexpr (DP > 0) {
                  const double* xr = s_ring + ((c0 + k0 + u - lane - 32 * r) & (RING - 1)) * XS;
                  double row[DP];
#pragma unroll
                  for (int c = 0; c < DP; ++c) row[c] = xr[c];
                  mx = fmax(mx, fabs(exact_dot<DP>(row, dy)));
                } else {
                  const int j = c0 + k0 + u - lane - 32 * r;
                  mx = fmax(mx, fabs(exact_dot_rows(xrows0 + static_cast<size_t>(j) * P.ld,
                                                    yrows0 + static_cast<size_t>(irow[r]) * P.ld, P.dim)));
                }
              }
          }
        }
      }
    }
  };
  // hand the chunk's top-row alpha' to the band above and publish progress
  auto hand_up = [&](int c0, int kend) {
    // hand the top row's alpha' of this chunk to the band above, then publish
    // progress every kPublish columns
    if (intra_out) {
      __syncwarp();  // lane 31's ring writes before lane 0's release
      if (lane == 0) st_release_cta_u32(&ctl->up_prod, static_cast<unsigned>(c0 + kend));
    } else if (has_above) {
      const int jfirst = c0 - 31 - 32 * (R - 1);
      const int pieces = direct_top_out(DP) ? 0 : kend * NP / 2;
      for (int e = lane; e < pieces; e += 32) {
        const int kk = e / (NP / 2);
        const int jj = jfirst + kk;
        if (jj >= 0 && jj < cols) {
          const double2 v = *reinterpret_cast<const double2*>(s_out + 2 * e);
          __stcg(reinterpret_cast<double2*>(out_buf + static_cast<size_t>(jj) * NP + (2 * e - kk * NP)), v);
        }
      }
      // columns handed up before / after this chunk
      const int done0 = min(max(jfirst, 0), cols);
      const int done1 = min(max(jfirst + kend, 0), cols);
      if (streaming && done1 > done0 && (done1 == cols || done1 / kPublish != done0 / kPublish)) {
        // bar.warp.sync orders every lane's column stores before lane 0's
        // release store (PTX memory model: barrier synchronisation is part
        // of causality order), so one release by one lane publishes them all
        // -- no per-lane fence.sc (MEMBAR.SC + L1 invalidation)
        __syncwarp();
        if (lane == 0) {
          if (xout)
            st_release_sys(out_prog, base + done1);  // peer-memory data before the peer-visible counter
          else
            st_release_gpu(out_prog, base + done1);
        }
      }
    }
  };

  // prefetch depth is one group, but only when its columns are already
  // published: a caught-up band (latency-bound chains) stages the group it
  // is about to run instead of waiting one group longer for the next one,
  // which would add a whole group to every band's hand-over lag
  int staged = c_begin;
  for (int c0 = c_begin * K, chunk = c_begin; c0 < steps && chunk < c_end; c0 += K, ++chunk) {
    __syncwarp();  // everyone is done with the buffers group chunk + 1 overwrites
    if (staged < chunk && chunk < ngroups && chunk < c_end) {
      if (gdep && !wait_progress(P, in_prog, base + min(cols, (chunk + 1) * K), seen, p, b, xin)) return kBandAbort;
      stage_group(chunk);
      staged = chunk;
    }
    if (chunk + 1 < ngroups && chunk + 1 < c_end &&
        (!gdep || poll_progress(in_prog, base + min(cols, (chunk + 2) * K), seen, xin))) {
      stage_group(chunk + 1);
      staged = chunk + 1;
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    if (intra_in && c0 < cols) {
      // columns [c0, c0 + K) of the band below: its top row's steps c0 + 31 ...
      const int cend = min(cols, c0 + K);
      const unsigned need = static_cast<unsigned>(cend + 31);
      if (!intra_wait(&below_ctl->up_prod, need)) return kBandAbort;
      double* dst = s_alpha + (chunk & 1) * kStage;
      const int pieces = (cend - c0) * NP / 2;
      for (int e = lane; e < pieces; e += 32) {
        const int kk = e / (NP / 2);
        const double* src = below_ring + ((c0 + kk + 31) & (kUpRing - 1)) * NP + (2 * e - kk * NP);
        *reinterpret_cast<double2*>(dst + 2 * e) = *reinterpret_cast<const double2*>(src);
      }
      __syncwarp();  // every lane's ring reads before lane 0 frees the steps
      if (lane == 0) st_release_cta_u32(&below_ctl->up_cons, need);
      __syncwarp();
    }
    if (intra_out) {
      // this chunk's top-row outputs go to ring chunk (chunk mod kUpChunks):
      // the band above must have copied the steps it held
      const int need = (chunk - kUpChunks + 1) * K;
      if (need > 0 && !intra_wait(&ctl->up_cons, static_cast<unsigned>(need))) return kBandAbort;
      s_out = up_ring + (chunk & (kUpChunks - 1)) * kStage;
    }
    const double* stage = s_alpha + (chunk & 1) * kStage;
    const double* dl = DP > 0 ? s_delta : s_tab + (chunk & 1) * K * 32;
    const int kend = min(K, steps - c0);
    if (DP == 0 && !tab_mode) {
      // the producers have written every column this chunk reads: < c0 + K
      // (columns at or past `cols` belong to finished rows and are not used)
      const unsigned need = static_cast<unsigned>((min(cols, c0 + K) + kRhoB - 1) / kRhoB);
      int stuck = 0;
      if (lane == 0 && ld_acquire_cta_u32(&ctl->prod) < need) {
        const unsigned long long t0 = globaltimer_ns();
#ifdef SK_RHO_PROFILE
        struct Acc {
          unsigned long long t0;
          unsigned long long* dst;
          __device__ ~Acc() { atomicAdd(dst, globaltimer_ns() - t0); }
        } acc_wait{t0, P.watchdog + 5};
#endif
        unsigned ns = 16;
        while (ld_acquire_cta_u32(&ctl->prod) < need) {
          __nanosleep(ns);
          if (ns < 256) ns *= 2;
          if (globaltimer_ns() - t0 > P.watchdog_ns) {
            if (atomicCAS(P.watchdog, 0ull, 1ull) == 0ull) {
              P.watchdog[1] = p;
              P.watchdog[2] = b;
              P.watchdog[3] = need;
              P.watchdog[4] = ctl->prod;
            }
            stuck = 1;
            break;
          }
        }
      }
      if (__shfl_sync(0xffffffffu, stuck, 0)) return kBandAbort;
      __syncwarp();  // lane 0's acquire before every lane reads the ring
    }
    form_deltas(c0, kend, dl);
    __syncwarp();
    auto run_chunk = [&](bool tot) {
      int k = 0;
#pragma unroll 1
      for (; k + 1 < kend; k += 2) {
        step(tot, c0 + k, k, stage, dl, roA, roB);
        step(tot, c0 + k + 1, k + 1, stage, dl, roB, roA);
      }
      if (k < kend) {
        step(tot, c0 + k, k, stage, dl, roA, roB);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int m = 0; m < NA; ++m) roA[r][m] = roB[r][m];
      }
    };
    // totals where the pair's final tile can fall (or everywhere, kFlagAllTotals)
    if constexpr (kLiteral) {
      run_chunk(true);
    } else {
      // lane t meets its diagonal tile (row0 + t, row0 + t) at step row0 + 2t
      const bool diag_chunk = EXTRAS && P.diag != nullptr && c0 <= row0 + 62 && c0 + K > row0;
      if (all_totals || diag_chunk || (band_top && c0 + K > cols - 1))
        run_chunk(true);
      else
        run_chunk(false);
    }
    if constexpr (EXACT && kInlineDelta) {
      // exact max|delta| (bit-identical to max_abs_rho): |fast - sequential|
      // <= dot_err, so only a lane whose largest fast |delta| of the chunk
      // plus dot_err reaches the running exact max can raise it -- rare once
      // the max has settled; that lane re-forms its chunk's products with the
      // sequential dot from the dx ring (the chunk's rows are still there: the
      // next chunk's staging fills rows 16 to 31 columns ahead of lane 31)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const bool cand = __longlong_as_double(static_cast<long long>(fmxb[r])) + P.dot_err >= mx;
        if (__any_sync(0xffffffffu, cand) && cand) {
#pragma unroll 1
          for (int k = 0; k < kend; ++k) {
            const int j = c0 + k - lane - 32 * r;
            if (row_ok[r] && j >= 0 && j < cols) {
              const double* xr = s_ring + (j & (RING - 1)) * XS;
              double row[DP > 0 ? DP : 1];
#pragma unroll
              for (int c = 0; c < DP; ++c) row[c] = xr[c];
              mx = fmax(mx, fabs(exact_dot<DP>(row, dyr[r])));
            }
          }
        }
        fmxb[r] = 0ull;
      }
    }
    hand_up(c0, kend);
    if (DP == 0 && !tab_mode) {
      __syncwarp();  // every lane's ring reads of this chunk are done
      if (lane == 0) st_release_cta_u32(&ctl->cons, static_cast<unsigned>(chunk + 1));
    }
  }
  if (streaming && !has_above && P.bands > 1) {
    // the last band publishes completion too: the slot's next pair (p + slots)
    // may only rewrite the column buffer once this band has read all of it
    cp_async_wait<0>();
    __syncwarp();
    if (lane == 0) st_release_gpu(prog_row + b, base + cols);
  }
  if (save) {
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < NA; ++m)
        if (NA <= kMaxRegOrder + 1 || m < n) rec[(r * NP + m) * 32 + lane] = roA[r][m];
    // the slots the unit's last step wrote (what the next step would read)
    const double* const spl = pass_in(static_cast<int>(min(static_cast<long long>(c_end) * K, static_cast<long long>(steps))));
    for (int e = lane; e < 32 * R * NP; e += 32) rec[32 * R * NP + e] = spl[e];
  }
  // per-pair error key (first failing tile) and max|delta|: min / max
  // reductions, so each segment flushes its part
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (jkey[r] != ~0u) atomicMin(P.err + out, err_key(irow[r], jkey[r] >> 2, jkey[r] & 3u));
  if constexpr (EXACT) {
    if (P.maxrho) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0 && mx > 0.0) {
        atomicMax(P.maxrho + out, static_cast<unsigned long long>(__double_as_longlong(mx)));
        if (P.maxrho_all) atomicMax(P.maxrho_all, static_cast<unsigned long long>(__double_as_longlong(mx)));
      }
    }
  }
  return kBandDone;
}

// ---- rho producer of a DP == 0 band CTA (warp 1): per unit, the band's
// rho for columns [c_lo, c_hi) in blocks of 32 rows x kRhoB columns.
// DMMA: rho = dY dX^T on the FP64 tensor cores, k staged through a
// kRhoStages-deep cp.async pipeline that runs on across block boundaries.
// EXACT_RHO (literal kernel): the reference's sequential non-FMA dot
// (wavefront.cpp:146-149), lane = row, so every delta is the reference's bits.
template <bool EXACT_RHO>
__device__ __forceinline__ void rho_producer(const SweepParams& P, double* __restrict__ ring,
                                             double* __restrict__ stg, RhoCtl* ctl, int lane, unsigned bar_start,
                                             unsigned bar_end) {
  constexpr int K = chunk_cols(1);
  constexpr int kStageSz = (32 + kRhoB) * kRhoKS;
  const int ld = P.ld;
  const int nk = (ld + kRhoKC - 1) / kRhoKC;
  for (;;) {
    named_bar_sync(bar_start, 64);  // the band's sweep warp published the unit (or stop)
    if (ctl->stop) return;
    const unsigned p = ctl->p, b = ctl->b;
    const int c_begin = ctl->c_begin;
    const long long c_end_cols = static_cast<long long>(ctl->c_end) * K;
    const int rows = P.rows, cols = P.cols;
    const int row0 = static_cast<int>(b) * 32;
    const int c_lo = max(0, c_begin * K - 31);
    const int c_hi = static_cast<int>(min(static_cast<long long>(cols), c_end_cols));
    const int q0 = c_lo / kRhoB, q1 = (c_hi + kRhoB - 1) / kRhoB;
    const int T = max(0, q1 - q0) * nk;
    const double* xs = P.xinc + P.pair_x[p] * P.sx + ld;  // column j's increments at xs + j * ld
    const double* ys = P.yinc + P.pair_y[p] * P.sy + ld;  // row i's at ys + i * ld
    // columns before 0 read delta = 0 (a tile's unit-series steps before its
    // first column); ring slots not yet produced are never read by live tiles
    for (int e = lane; e < kRhoW * 32; e += 32) ring[e] = 0.0;
    auto load = [&](int t) {
      if (t < T) {
        const int q = q0 + t / nk, k0 = (t - (t / nk) * nk) * kRhoKC;
        double* A = stg + (t % kRhoStages) * kStageSz;
        for (int e = lane; e < (32 + kRhoB) * (kRhoKC / 2); e += 32) {
          const int r = e / (kRhoKC / 2), c = (e - r * (kRhoKC / 2)) * 2;
          const int k = k0 + c;
          const bool is_a = r < 32;
          const int idx = is_a ? row0 + r : q * kRhoB + (r - 32);
          const bool ok = (is_a ? idx < rows : idx < cols) && k < ld;
          const double* src = (is_a ? ys : xs) + static_cast<size_t>(ok ? idx : 0) * ld + (ok ? k : 0);
          cp_async_16_zfill(A + r * kRhoKS + c, src, ok);
        }
      }
      cp_async_commit();
    };
#ifdef SK_RHO_PROFILE
    const unsigned long long tu = globaltimer_ns();
#endif
#pragma unroll
    for (int t = 0; t < kRhoStages - 1; ++t) load(t);
    double acc[EXACT_RHO ? 32 : 4 * 4 * 2];
#pragma unroll
    for (int e = 0; e < (EXACT_RHO ? 32 : 32); ++e) acc[e] = 0.0;
    bool aborted = false;
    for (int t = 0; t < T; ++t) {
      cp_async_wait<kRhoStages - 2>();
      __syncwarp();
      const double* A = stg + (t % kRhoStages) * kStageSz;
      const double* Bm = A + 32 * kRhoKS;
      if constexpr (EXACT_RHO) {
        // lane = row; 32 sequential dots, one per column of the block
#pragma unroll 1
        for (int k = 0; k < kRhoKC; ++k) {
          const double av = A[lane * kRhoKS + k];
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(av, Bm[c * kRhoKS + k]));
        }
      } else {
#pragma unroll
        for (int k4 = 0; k4 < kRhoKC; k4 += 4) {
          double a[4], bb[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            a[m] = A[(m * 8 + (lane >> 2)) * kRhoKS + k4 + (lane & 3)];
            bb[m] = Bm[(m * 8 + (lane >> 2)) * kRhoKS + k4 + (lane & 3)];
          }
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              double (&c2)[2] = *reinterpret_cast<double (*)[2]>(&acc[(mt * 4 + nt) * 2]);
              dmma_884(c2, a[mt], bb[nt]);
            }
        }
      }
      __syncwarp();  // the stage is read before it is refilled
      load(t + kRhoStages - 1);
      if (t - (t / nk) * nk == nk - 1) {
        // block q done: wait until the consumer has left the ring slot
        // (columns < (q - RB + 1) B are last read at step column + 31)
        const int q = q0 + t / nk;
        const long long need = static_cast<long long>(q - kRhoRB + 1) * kRhoB + 31;
        int stop = 0;
        if (lane == 0) {
          unsigned ns = 32;
#ifdef SK_RHO_PROFILE
          const unsigned long long tw = globaltimer_ns();
#endif
          while (static_cast<long long>(ld_acquire_cta_u32(&ctl->cons)) * K < need) {
            if (*reinterpret_cast<volatile unsigned*>(&ctl->abort)) {
              stop = 1;
              break;
            }
            __nanosleep(ns);
            if (ns < 512) ns *= 2;
          }
#ifdef SK_RHO_PROFILE
          atomicAdd(P.watchdog + 6, globaltimer_ns() - tw);
#endif
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) {
          aborted = true;
          break;
        }
        __syncwarp();
        const int cbase = q * kRhoB;
        if constexpr (EXACT_RHO) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            ring[((cbase + c) & (kRhoW - 1)) * 32 + lane] = acc[c];
            acc[c] = 0.0;
          }
        } else {
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int row = mt * 8 + (lane >> 2), col = nt * 8 + 2 * (lane & 3) + e;
                ring[((cbase + col) & (kRhoW - 1)) * 32 + row] = acc[(mt * 4 + nt) * 2 + e];
                acc[(mt * 4 + nt) * 2 + e] = 0.0;
              }
        }
        __syncwarp();  // every lane's ring stores before lane 0 publishes them
        if (lane == 0) st_release_cta_u32(&ctl->prod, static_cast<unsigned>(q + 1));
      }
    }
    (void)aborted;
#ifdef SK_RHO_PROFILE
    if (lane == 0) atomicAdd(P.watchdog + 7, globaltimer_ns() - tu);
#endif
    cp_async_wait<0>();
    __syncwarp();
    named_bar_sync(bar_end, 64);  // the sweep warp finished the unit
  }
}

// Persistent: grid = resident CTAs; dynamic shared memory =
// sweep_smem_doubles(N, DP) doubles.  DP == 0: warps 0..B-1 sweep B bands,
// warps B..2B-1 produce their rho (band slot k: sweep warp k, producer warp
// B + k, named barriers 1 + 2k / 2 + 2k), B = rho_bands(N).
template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
__global__ void __launch_bounds__(sweep_warps(N, DP) * 32, DP == 0 || LIT ? 1 : sweep_min_blocks(N))
    sweep_kernel(const SweepParams P) {
  constexpr int kBands = DP == 0 ? rho_bands(N) : 1;
  static_assert(DP > 0 || kBands >= 1, "a band's shared memory must fit the SM");
  extern __shared__ __align__(16) double s_dyn[];
  __shared__ RhoCtl s_ctls[kBands];
  __shared__ unsigned s_claim;  // intra: the CTA's first unit of this round
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int kslot = DP == 0 ? warp % kBands : 0;
  RhoCtl& s_ctl = s_ctls[kslot];
  const unsigned bar_start = 1u + 2u * kslot, bar_end = 2u + 2u * kslot;
  double* smem = DP == 0 ? s_dyn + kslot * (P.slot_stride > 0 ? P.slot_stride : rho_slot_doubles(N))
                         : s_dyn + warp * stage_doubles_per_warp(N, DP, LIT);
  if constexpr (DP == 0) {
    if (warp >= kBands) {
      if (P.rho_tab != nullptr) return;  // table mode: no producers
      double* ring = smem + stage_doubles_per_warp(N, 0);
      rho_producer<N == 0 || LIT>(P, ring, ring + rho_ring_doubles(), &s_ctl, lane, bar_start, bar_end);
      return;
    }
  }
  constexpr int H = 32 * rows_per_lane(N);
  constexpr int K = chunk_cols(rows_per_lane(N));
  // bands of each pair this launch sweeps (all, or this GPU's strip blocks)
  const unsigned nb = static_cast<unsigned>(P.units_pair_streaming);
  const unsigned gsz = static_cast<unsigned>(P.group) * nb;
  // one unit; DP == 0: hand it to the producer warp first, and meet it again
  // at the end (the ring is reused by the next unit)
  const bool with_producer = DP == 0 && P.rho_tab == nullptr;
  auto run_unit = [&](unsigned p, unsigned b, int c_begin, int c_end, bool restore, bool save) {
    if (with_producer) {
      if (lane == 0) {
        s_ctl.p = p;
        s_ctl.b = b;
        s_ctl.c_begin = c_begin;
        s_ctl.c_end = c_end;
        s_ctl.stop = 0u;
        s_ctl.abort = 0u;
        s_ctl.prod = static_cast<unsigned>(max(0, c_begin * K - 31) / kRhoB);
        s_ctl.cons = static_cast<unsigned>(c_begin);
      }
      named_bar_sync(bar_start, 64);
    }
    const int st = sweep_band<N, DP, EXACT, EXTRAS, LIT>(P, p, b, lane, smem, c_begin, c_end, restore, save, &s_ctl);
    if (with_producer) {
      if (st == kBandAbort && lane == 0) *reinterpret_cast<volatile unsigned*>(&s_ctl.abort) = 1u;
      named_bar_sync(bar_end, 64);
    }
    return st;
  };
  for (;;) {
    unsigned p, b;
    int c_begin = 0, c_end = 0x7fffffff, seg = 0;
    SegRange sr{0, 0};
    bool restore = false, save = false;
    if (P.seg_cols == 0) {
      // streaming: static unit order (group g, band b, pair q within the group)
      unsigned u = 0;
      const unsigned total = static_cast<unsigned>(P.npairs) * nb;
      if (DP == 0 && N > 0 && P.intra) {
        // one round per CTA: its sweep warps meet, warp 0 claims kBands
        // consecutive units (consecutive bands of one pair), warp w takes the
        // w-th; the decision to stop is the same for every warp
        named_bar_sync(kIntraBar, kBands * 32);
        if (warp == 0 && lane == 0)
          s_claim = *reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0
                        ? ~0u
                        : atomicAdd(P.queue, static_cast<unsigned>(kBands));
        if (lane == 0) {
          s_ctl.up_prod = 0u;
          s_ctl.up_cons = 0u;
        }
        named_bar_sync(kIntraBar, kBands * 32);
        const unsigned c0 = *reinterpret_cast<volatile unsigned*>(&s_claim);
        if (c0 == ~0u || c0 >= total) break;
        u = c0 + static_cast<unsigned>(kslot);
        if (u >= total) continue;  // no unit this round; the next claim ends the loop
      } else {
        if (lane == 0) u = atomicAdd(P.queue, 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= total) break;
        if (*reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0) break;
      }
      const unsigned g = u / gsz;
      const unsigned rem = u - g * gsz;
      const unsigned g0 = g * static_cast<unsigned>(P.group);
      const unsigned gcount = min(static_cast<unsigned>(P.group), static_cast<unsigned>(P.npairs) - g0);
      const unsigned bi = rem / gcount;  // the pair's bi-th band of this launch
      p = g0 + (rem - bi * gcount);
      // strips: bi-th band of the blocks xrank, xrank + xgpus, ...
      const unsigned S = static_cast<unsigned>(P.xblock);
      b = P.xemul ? bi : (static_cast<unsigned>(P.xrank) + static_cast<unsigned>(P.xgpus) * (bi / S)) * S + bi % S;
    } else {
      // segment DAG: claim the next cell of the ready list, wait for its unit
      unsigned u = 0;
      if (lane == 0) {
        const unsigned h = atomicAdd(P.ctr, 1u);
        if (h >= P.units_total) {
          u = ~0u;
        } else {
          const unsigned* cell = P.rq + h;
          unsigned v, ns = 32;
          const unsigned long long t0 = globaltimer_ns();
          for (unsigned it = 1; (v = ld_acquire_u32(cell)) == 0u; ++it) {
            __nanosleep(ns);
            if (ns < 1024) ns *= 2;
            if ((it & 63) == 0) {
              if (*reinterpret_cast<volatile unsigned long long*>(P.watchdog) != 0) {
                v = 0u;
                break;
              }
              if (globaltimer_ns() - t0 > P.watchdog_ns) {
                if (atomicCAS(P.watchdog, 0ull, 1ull) == 0ull) {
                  P.watchdog[1] = ~0ull;
                  P.watchdog[2] = ~0ull;
                  P.watchdog[3] = h;
                  P.watchdog[4] = ld_relaxed_u32(P.ctr + kCtrLine);
                }
                v = 0u;
                break;
              }
            }
          }
          u = v - 1u;  // ~0u on abort
        }
      }
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u == ~0u) break;
      __syncwarp();  // lane 0's acquire of the unit before every lane reads its inputs
      const unsigned spb = static_cast<unsigned>(P.segs_per_band);
      const unsigned pb = u / spb;
      p = pb / static_cast<unsigned>(P.bands);
      b = pb - p * static_cast<unsigned>(P.bands);
      sr = seg_range(P.rows, P.cols, static_cast<int>(b), H, P.seg_cols);
      seg = sr.lo + static_cast<int>(u - pb * spb);
      // steps [seg L - b H, (seg+1) L - b H) clipped to the band: chunk range
      c_begin = max(0, seg * P.seg_cols - static_cast<int>(b) * H) / K;
      c_end = ((seg + 1) * P.seg_cols - static_cast<int>(b) * H) / K;
      restore = seg > sr.lo;
      save = seg < sr.hi;
    }
#ifdef SK_PROFILE_WAITS
    const long long t0 = clock64();
    const unsigned long long gt0 = globaltimer_ns();
    const unsigned wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) g_wwait[wid] = 0;
    const int st = run_unit(p, b, c_begin, c_end, restore, save);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(P.watchdog + 7), clock64() - t0);
      const unsigned t = atomicAdd(&g_tidx, 1u);
      if (t < kTraceUnits) {
        unsigned smid, hwwarp;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(hwwarp));
        smid |= hwwarp << 8;
        g_utrace[4 * t] = p | (static_cast<unsigned long long>(b) << 20) | (static_cast<unsigned long long>(smid) << 40);
        g_utrace[4 * t + 1] = gt0;
        g_utrace[4 * t + 2] = globaltimer_ns();
        g_utrace[4 * t + 3] = g_wwait[wid] | (static_cast<unsigned long long>(seg) << 40);
      }
    }
#else
    const int st = run_unit(p, b, c_begin, c_end, restore, save);
#endif
    if (st == kBandAbort) {
      if (DP == 0 && N > 0 && P.intra && P.seg_cols == 0) continue;  // the siblings meet at the next round (watchdog set)
      break;
    }
    if (P.seg_cols > 0) {
      __syncwarp();  // every lane's outputs before lane 0 releases them
      if (lane == 0) {
        const unsigned spb = static_cast<unsigned>(P.segs_per_band);
        const unsigned slot = p % static_cast<unsigned>(P.slots);
        const size_t slot_base = static_cast<size_t>(slot) * P.bands * spb;
        const unsigned unit_base = p * static_cast<unsigned>(P.bands) * spb;
        // right neighbour (b, seg + 1): inputs (b, seg) and (b - 1, seg + 1)
        if (seg < sr.hi) {
          const SegRange below = b > 0 ? seg_range(P.rows, P.cols, static_cast<int>(b) - 1, H, P.seg_cols) : SegRange{0, -1};
          const unsigned nd = 1u + (b > 0 && seg + 1 <= below.hi ? 1u : 0u);
          const unsigned off = b * spb + static_cast<unsigned>(seg + 1 - sr.lo);
          dep_arrive(P, slot_base + off, nd, unit_base + off);
        }
        // the unit above that this one completes: (b + 1, seg), or -- from the
        // band's last segment, when band b + 1 starts later (one-column pairs)
        // -- band b + 1's first segment; inputs: its left neighbour (if any)
        // and this unit
        if (b + 1 < static_cast<unsigned>(P.bands)) {
          const SegRange above = seg_range(P.rows, P.cols, static_cast<int>(b) + 1, H, P.seg_cols);
          const int tgt = seg == sr.hi ? max(seg, above.lo) : seg;
          if (tgt >= above.lo) {
            const unsigned nd = 1u + (tgt > above.lo ? 1u : 0u);
            const unsigned off = (b + 1) * spb + static_cast<unsigned>(tgt - above.lo);
            dep_arrive(P, slot_base + off, nd, unit_base + off);
          }
        }
        // the pair's last unit: every other unit of the pair is done (all are
        // its ancestors) -- recycle the slot's counters, queue the next pair
        const bool last = b + 1 == static_cast<unsigned>(P.bands) && seg == sr.hi;
        if (last && p + P.slots < static_cast<unsigned>(P.npairs)) {
          for (size_t k = 0; k < static_cast<size_t>(P.bands) * spb; ++k) P.dep[slot_base + k] = 0u;
          rq_push(P, (p + P.slots) * static_cast<unsigned>(P.bands) * spb);
        }
        atomicAdd(P.ctr + 2 * kCtrLine, 1u);
      }
    }
  }
  if (with_producer) {
    if (lane == 0) s_ctl.stop = 1u;
    named_bar_sync(bar_start, 64);  // releases the band slot's producer
  }
}

}  // namespace skb
