/*
 * sigker_b200.h -- the C-ABI drop-in boundary of the B200 tile solver.
 *
 * Plain pointers and sizes only (no torch / CUDA types).  Every entry point
 * replaces one reference interface of `sigker` (/root/reference/proj) and
 * keeps its argument meaning and error behaviour; the C++ layer
 * (include/sigker/*.hpp, paper_2502_20392_b200/host/) maps the status codes
 * back to the reference's exception types.  INTEGRATION.md shows the
 * bindings (C++ API, ctypes) a maintainer adds.
 *
 * Layout conventions (the reference's, time_series.hpp:10-38):
 *   a series of length L and dimension d is L*d doubles, row-major
 *   (one sample point per row); tile (i, j) has j along the FIRST series x
 *   (columns, cols = lx-1) and i along the SECOND series y (rows = ly-1).
 *
 * Threading: all entry points are reentrant.  Each calling host thread owns
 * its own CUDA stream and device workspace (reference requirement: gram.cpp
 * calls propagate concurrently from pool workers), there is no global
 * device lock.  There is no CPU fallback: without a CUDA device every
 * compute entry point returns SK_CUDA_ERROR.
 */
#ifndef SIGKER_B200_H
#define SIGKER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 3

/* Status codes (errors.hpp:10-53 of the reference). */
enum sk_code {
  SK_OK = 0,
  SK_INVALID_ARGUMENT = 1,      /* std::invalid_argument                         */
  SK_NUMERIC_OVERFLOW = 2,      /* sigker::NumericOverflowError (tile_k, tile_l) */
  SK_INCONSISTENT_BOUNDARY = 3, /* sigker::InconsistentBoundaryError             */
  SK_INTERNAL = 4,              /* any other failure                             */
  SK_CUDA_ERROR = 5             /* no device / launch failure / out of memory    */
};

typedef struct sk_status {
  int32_t code;
  uint64_t tile_k; /* 1-based tile index along the first series (k = j + 1)  */
  uint64_t tile_l; /* 1-based tile index along the second series (l = i + 1) */
  char message[256];
} sk_status;

/* flags */
#define SK_STRICT_CORNER 1u /* reference corner check, tile_series.cpp:70-75 (C++ API default) */
#define SK_W_FAULT 4u       /* negative control: flip W[1][1], tile_series.cpp:51-52           */

int sk_abi_version(void);
/* Number of visible CUDA devices (0 when none). */
int sk_device_count(void);
/* Device used by the calling thread's context (default 0). */
int sk_set_device(int device, sk_status* st);
/* Route the calling thread's work onto an existing cudaStream_t (NULL =
 * the library's own stream).  Lets a caller time the work with its own
 * events on that stream. */
int sk_set_stream(void* cuda_stream, sk_status* st);

/* wavefront.hpp:41-47 propagate / propagate_grid (wavefront.cpp:70-199).
 * order in [1, 64].  value <- K(1,1); peak_live <- the reference's
 * peak_live_series; grid (lx*ly, may be NULL) <- K at every knot pair,
 * entry [a*ly + b]; diag (min(lx,ly)-1 entries, may be NULL) <- K at knots
 * (i+1, i+1). */
int sk_propagate(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                 uint32_t flags, double* value, uint64_t* peak_live, double* grid, double* diag,
                 sk_status* st);

/* time_series.hpp:57 IncrementTable::max_abs_rho (time_series.cpp:64-73),
 * bit-identical (sequential non-FMA products). */
int sk_max_abs_rho(const double* x, size_t lx, const double* y, size_t ly, size_t dim, double* out,
                   sk_status* st);

/* truncation.hpp:36 estimate_order (truncation.cpp:41-55); host arithmetic. */
int sk_estimate_order(double max_abs_rho, size_t length, double tol, int* order, int* converged,
                      sk_status* st);

/* wavefront.hpp:58-60 step_tile (wavefront.cpp:223-237): one tile on the
 * device with the reference's exact arithmetic (bit-identical).  order in
 * [0, 64]; series hold order+1 coefficients.  total may be NULL. */
int sk_step_tile(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                 double* out_beta, double* total, sk_status* st);

/* Diagnostics: the same tile through the factorial-scaled register solver
 * used by the sweep for order <= 16 (not bit-identical). */
int sk_step_tile_fast(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                      double* out_beta, double* total, sk_status* st);

/* Batched independent pairs (addition the reference lacks; per pair exactly
 * propagate_with_policy, wavefront.cpp:206-221).  Pair k is
 * (xs + k*lx*dim, ys + k*ly*dim).  adaptive != 0: per-pair order from
 * estimate_order(max|rho|, tol); else `order` for every pair.
 * Outputs (npairs entries each; any may be NULL except values):
 *   values, orders, converged, max_abs_rho (exact, only when adaptive),
 *   per_pair status.  Return value: SK_OK unless the call itself failed
 *   (bad arguments / device error); per-pair numeric failures leave NaN in
 *   values and are reported in per_pair. */
int sk_pairwise(const double* xs, size_t lx, const double* ys, size_t ly, size_t npairs, size_t dim,
                int adaptive, int order, double tol, uint32_t flags, double* values, int* orders,
                int* converged, double* max_abs_rho, sk_status* per_pair, sk_status* st);

/* Same with device-resident inputs d_xs, d_ys and device output d_values
 * (already allocated by the caller, e.g. torch tensors); host outputs as
 * above.  Work is issued on the thread's stream (sk_set_stream). */
int sk_pairwise_device(const double* d_xs, size_t lx, const double* d_ys, size_t ly, size_t npairs,
                       size_t dim, int adaptive, int order, double tol, uint32_t flags, double* d_values,
                       int* orders, int* converged, sk_status* per_pair, sk_status* st);

/* gram.hpp:46 gram_matrix (gram.cpp:16-98) over a family of m series of the
 * common length len (the caller pads, gram.cpp:17-27).  Upper-triangle pairs
 * (i <= j) in row-major order are split into nshards contiguous equal-work
 * ranges; this call evaluates shard `shard` (nshards = 1: everything) and
 * writes mirrored entries of values/orders (m*m; untouched entries are NaN /
 * 0).  scan_products != 0 (adaptive or compute_bound): pair_max (m*m, may be
 * NULL) receives each pair's exact max|rho| and *max_product their maximum.
 * Entries that raise NumericOverflowError are NaN and counted in
 * *n_failures; their records come from sk_gram_failures.  Any other
 * per-entry failure (InconsistentBoundaryError) is returned as the call's
 * status, as gram.cpp:74-77 only catches overflow.
 * converged <- 0 if any adaptive search saturated. */
int sk_gram(const double* family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
            uint32_t flags, int scan_products, size_t shard, size_t nshards, double* values, int* orders,
            double* pair_max, double* max_product, int* converged, size_t* n_failures, sk_status* st);

/* The same on a device-resident family (d_family: m*len*dim doubles in this
 * thread's device memory) for the upper-triangle pair range [first, last)
 * (row-major, 0 <= first <= last <= m(m+1)/2): each pair's value -- NaN for
 * an overflow entry -- goes into both mirrored cells of the device matrix
 * d_matrix (m*m doubles); other cells are not touched.  Work is issued on
 * the thread's stream (sk_set_stream); the call returns when it is done. */
int sk_gram_device(const double* d_family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
                   uint32_t flags, int scan_products, size_t first, size_t last, double* d_matrix,
                   double* max_product, int* converged, size_t* n_failures, sk_status* st);

/* One overflow entry of the calling thread's last sk_gram / sk_gram_device
 * call (gram.hpp:20-24 GramEntryError).  sk_gram_failures copies up to cap
 * records in (row, col) row-major order and returns how many it copied. */
typedef struct sk_gram_failure {
  uint32_t row, col; /* row <= col */
  sk_status status;
} sk_gram_failure;
size_t sk_gram_failures(sk_gram_failure* out, size_t cap);

/* Row-major upper-triangle pair indices [first, last) that shard `shard` of
 * `nshards` evaluates in sk_gram (equal pair counts; pairs cost the same
 * because the family is padded to one length).  Host arithmetic only. */
int sk_gram_shard_range(size_t m, size_t shard, size_t nshards, size_t* first, size_t* last);

/* 1 when every one of the n doubles is finite, else 0 (the TimeSeries
 * constructor's check, time_series.cpp:9-19): a branch-free exponent test,
 * split over host threads for large inputs.  Host memory, host work only. */
int sk_all_finite(const double* v, size_t n);

/* ---- Multi-GPU long pair: block-cyclic strips (cfg 3).
 * The ly-1 tile rows are cut into 32-row bands (sk_strip_bands), the bands
 * into blocks of `block` bands, and the blocks are dealt round-robin over the
 * GPUs: GPU g sweeps blocks g, g+G, g+2G, ... (rounds r = 0, 1, ...), all in
 * one persistent launch.  At every block boundary the top band of block k
 * streams its alpha series into the exchange area of the GPU of block k+1
 * (peer stores over NVLink, system-scope release / acquire on a progress
 * counter; GPU G-1 hands to GPU 0).  Contiguous strips (round 1) starve: a
 * GPU's top band starts only after its whole strip has swept twice
 * (tools/strip_sim.py).  Setup: every GPU allocates its exchange area with
 * in_rounds of sk_strip_plan (sk_exchange_alloc) and exports it
 * (sk_ipc_handle); the previous GPU maps it (sk_ipc_open).  All GPUs of the
 * pair run concurrently.  Exchange areas hold `rounds` slots of (lx-1) x
 * (order+1, even) doubles and `rounds` progress counters (128 B apart). */
int sk_strip_bands(size_t ly, int order, size_t* bands);
int sk_strip_plan(size_t ly, int order, size_t gpus, size_t rank, size_t block, size_t* owned_bands,
                  size_t* rounds, size_t* in_rounds);
int sk_exchange_alloc(size_t lx, int order, size_t rounds, void** abuf, void** prog, sk_status* st);
int sk_exchange_reset(void* prog, size_t rounds, sk_status* st);
int sk_exchange_free(void* abuf, void* prog);
int sk_ipc_handle(void* dptr, void* handle64, sk_status* st);
int sk_ipc_open(const void* handle64, void** dptr, sk_status* st);
int sk_ipc_close(void* dptr);
/* One process driving several GPUs: enable the calling thread's device to
 * access `peer`'s memory, then pass exchange buffers as plain pointers. */
int sk_enable_peer_access(int peer, sk_status* st);
int sk_propagate_strip(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                       uint32_t flags, size_t gpus, size_t rank, size_t block, const void* in_abuf,
                       const void* in_prog, void* out_abuf, void* out_prog, double* value, double* diag,
                       sk_status* st);
/* One-GPU emulation of the whole pipeline of `gpus` GPUs in a single launch
 * (every band, global order; column buffers and exchange areas per virtual
 * GPU; every `block` bands the hand-off goes through an exchange area with the
 * multi-GPU protocol, the last virtual GPU handing to the first).  Test entry
 * point. */
int sk_propagate_split(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                       uint32_t flags, size_t gpus, size_t block, double* value, sk_status* st);

/* Device-time accounting of the sweep kernels on the calling thread
 * (CUDA events around every sweep launch). */
typedef struct sk_stats {
  uint64_t sweep_launches; /* tile-sweep kernel launches                  */
  uint64_t aux_launches;   /* other kernels (increments, scans, tables)   */
  double sweep_ms;         /* summed device time of the sweep launches    */
  double tiles;            /* tile-updates processed by those launches    */
  double tile_flops;       /* algorithmic FP64 flops, sum of F(N,d) per tile */
  uint64_t literal_rechecks; /* strict corner: pairs re-swept with the literal kernel (ABI 3) */
} sk_stats;

int sk_stats_enable(int enable);
int sk_stats_reset(void);
int sk_stats_get(sk_stats* out);

/* Free the calling thread's device workspace. */
int sk_release(void);

#ifdef __cplusplus
}
#endif

#endif /* SIGKER_B200_H */
