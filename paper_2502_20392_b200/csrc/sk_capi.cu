// The C-ABI (include/sigker_b200.h): host orchestration of the B200 path.
//
// Per call: H2D of the series -> increments kernel (K1) -> order pre-pass
// (Cauchy-Schwarz bound, exact max|rho| scan only where the bound cannot
// prove the order) -> one persistent banded sweep launch per distinct order
// (K2 + K3 fused) -> D2H of values / error keys / max|rho|.
// Per host thread: one context = device, stream, grow-only workspace.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <vector>
#include <thread>

#include <chrono>
#include <cstdlib>

#include "sigker_b200.h"
#include "sk_internal.h"
#include "sk_sweep.cuh"

namespace {

using namespace skb;

// ------------------------------------------------------------------ status
int set_status(sk_status* st, int code, uint64_t k, uint64_t l, const char* fmt, ...) {
  if (st) {
    st->code = code;
    st->tile_k = k;
    st->tile_l = l;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(st->message, sizeof st->message, fmt, ap);
    va_end(ap);
  }
  return code;
}

void clear_status(sk_status* st) {
  if (st) std::memset(st, 0, sizeof *st);
}

int cuda_fail(sk_status* st, cudaError_t e, const char* where) {
  return set_status(st, SK_CUDA_ERROR, 0, 0, "%s: %s", where, cudaGetErrorString(e));
}

#define SK_CUDA(call)                                       \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(st, e_, #call); \
  } while (0)

// ----------------------------------------------------------------- tracing
// SK_TRACE=1: host wall-clock per phase on stderr (diagnostics only).
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("SK_TRACE");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}
struct Tracer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!trace_on()) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sk] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// ------------------------------------------------------------ host tables
const double* host_factorials() {
  static double fact[171];
  static bool ready = false;
  if (!ready) {
    fact[0] = 1.0;
    for (int k = 1; k < 171; ++k) fact[k] = fact[k - 1] * static_cast<double>(k);  // tile_series.cpp:19-27
    ready = true;
  }
  return fact;
}

// truncation.cpp:41-55 at unit boundaries (tile_series.cpp:123-132 entry
// expression c = B * (A * W)); identical floating-point operations.
int host_estimate_order(double rho, double tol, int* order, int* converged) {
  const double* fact = host_factorials();
  for (int n = 8; n <= kMaxOrder; ++n) {
    double pw[kMaxOrder + 1];
    pw[0] = 1.0;
    for (int m = 1; m <= n; ++m) pw[m] = pw[m - 1] * rho;
    double tail = 0.0;
    for (int j = 0; j <= n; ++j) {
      const double b = (j == n) ? 1.0 : 0.0;
      const int lo = j < n ? j : n, hi = j < n ? n : j;
      tail += b * (pw[lo] * (fact[hi - lo] / (fact[hi] * fact[lo])));
    }
    for (int i = 0; i <= n; ++i) {
      const double b = (i == n) ? 1.0 : 0.0;
      const int lo = i < n ? i : n, hi = i < n ? n : i;
      tail += b * (pw[lo] * (fact[hi - lo] / (fact[hi] * fact[lo])));
    }
    if (tail < tol) {
      *order = n;
      *converged = 1;
      return SK_OK;
    }
  }
  *order = kMaxOrder;
  *converged = 0;
  return SK_OK;
}

// wavefront.cpp:19-30,107,111-125,175-176 -- the 1-thread live-series
// counter in closed form: the count only rises in prefill_units, and inside a
// diagonal every tile does sub(2) then add(up + right <= 2), so the peak is
// reached right after a prefill.  With m = min(rows, cols): diagonals
// 0..m-2 each prefill both edges (+2, nothing retires yet), reaching 2m; if
// the longer edge keeps going, diagonal m-1 prefills it once more (+1) before
// the shorter edge's retirements balance each later prefill.  Checked
// against the diagonal-by-diagonal count in tests/test_host.py.
uint64_t peak_live_closed_form(uint64_t rows, uint64_t cols) {
  const uint64_t m = std::min(rows, cols), big = std::max(rows, cols);
  return 2 * m + (big > m ? 1 : 0);
}

// ----------------------------------------------------------------- context
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) {
      cudaFree(p);
      p = nullptr;
      cap = 0;
    }
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return e;
    }
    cap = want;
    return cudaSuccess;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct StatRec {
  cudaEvent_t a, b;
  double tiles, flops;
};

struct Ctx {
  int device = 0;
  bool ready = false;
  cudaStream_t own = nullptr;
  cudaStream_t user = nullptr;
  int sms = 148;
  DevBuf raw_x, raw_y, xinc, yinc, sqn, pairs, values, err, maxr, prog, queue, abuf, tab, grid, diag, w65, tile_io,
      scan, wd, susp, dep, rq, redo, redo_out, gpairs, maxall;
  bool stats_on = false;
  std::vector<StatRec> stats;
  std::vector<sk_gram_failure> failures;  // the last sk_gram / sk_gram_device call's entry failures
  // host-side caches: cudaMemGetInfo can take milliseconds (driver round
  // trip), occupancy queries are per kernel variant and never change
  size_t free_cache = 0;
  int free_age = 0;
  std::map<int, int> occupancy;
  uint64_t sweep_launches = 0, aux_launches = 0, literal_rechecks = 0;
  double done_ms = 0.0, done_tiles = 0.0, done_flops = 0.0;

  // pinned staging for large pageable uploads (h2d): two buffers per worker
  std::vector<void*> stage;
  std::vector<cudaEvent_t> stage_ev;

  // cfg-4 overlap: the rho GEMM runs on `side` beside the sweep on stream()
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevBuf rowdone;  // per pair and 64-row block: GEMM tiles written

  cudaStream_t stream() const { return user ? user : own; }
  int ensure_side() {
    if (side && ev_fork && ev_join) return 0;  // (a partial failure retries the missing pieces)
    int prio_lo = 0, prio_hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) != cudaSuccess) return 1;
    if (!side && cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, prio_lo) != cudaSuccess) {
      side = nullptr;
      cudaGetLastError();  // the overlap is skipped; later launches must not see this error
      return 1;
    }
    if (!ev_fork && cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess) {
      ev_fork = nullptr;
      cudaGetLastError();  // the overlap is skipped; later launches must not see this error
      return 1;
    }
    if (!ev_join && cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess) {
      ev_join = nullptr;
      cudaGetLastError();  // the overlap is skipped; later launches must not see this error
      return 1;
    }
    return 0;
  }
  ~Ctx() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    rowdone.release();
    for (void* p : stage) cudaFreeHost(p);
    for (cudaEvent_t e : stage_ev) cudaEventDestroy(e);
    for (auto& r : stats) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    DevBuf* all[] = {&raw_x, &raw_y, &xinc, &yinc, &sqn, &pairs, &values, &err, &maxr,
                     &prog,  &queue, &abuf, &tab, &grid, &diag, &w65,   &tile_io, &scan, &wd,
                     &susp,  &dep,   &rq,   &redo, &redo_out, &gpairs, &maxall};
    for (DevBuf* b : all) b->release();
    if (own) cudaStreamDestroy(own);
  }
};

thread_local std::unique_ptr<Ctx> t_ctx;
thread_local int t_device = 0;

int get_ctx(Ctx** out, sk_status* st) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return set_status(st, SK_CUDA_ERROR, 0, 0,
                      "no CUDA device available (the B200 path has no CPU fallback): %s",
                      e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
  }
  if (t_ctx && t_ctx->device != t_device) t_ctx.reset();
  if (!t_ctx) {
    auto c = std::make_unique<Ctx>();
    c->device = t_device;
    SK_CUDA(cudaSetDevice(c->device));
    // the library's stream at the highest priority: where a launch runs a
    // helper kernel beside it (the cfg-4 GEMM on `side`), its CTAs are
    // dispatched first
    int prio_lo = 0, prio_hi = 0;
    SK_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SK_CUDA(cudaStreamCreateWithPriority(&c->own, cudaStreamNonBlocking, prio_hi));
    SK_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device));
    // W table, row stride 65 (tile_series.cpp:41-53 build_W_into)
    const double* fact = host_factorials();
    std::vector<double> w((kMaxOrder + 1) * (kMaxOrder + 1));
    for (int i = 0; i <= kMaxOrder; ++i)
      for (int j = i; j <= kMaxOrder; ++j) {
        const double v = fact[j - i] / (fact[j] * fact[i]);
        w[i * (kMaxOrder + 1) + j] = v;
        w[j * (kMaxOrder + 1) + i] = v;
      }
    // second copy with the negative-control flip of W[1][1] (tile_series.cpp:51-52)
    std::vector<double> wf(w);
    wf[1 * (kMaxOrder + 1) + 1] = -wf[1 * (kMaxOrder + 1) + 1];
    SK_CUDA(c->w65.ensure(2 * w.size() * sizeof(double)));
    SK_CUDA(cudaMemcpy(c->w65.p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
    SK_CUDA(cudaMemcpy(c->w65.as<double>() + w.size(), wf.data(), w.size() * sizeof(double),
                       cudaMemcpyHostToDevice));
    c->ready = true;
    t_ctx = std::move(c);
  }
  SK_CUDA(cudaSetDevice(t_ctx->device));
  *out = t_ctx.get();
  return SK_OK;
}

// --------------------------------------------------------------- sweeps
struct PairSet {
  const double* d_xinc;
  const double* d_yinc;
  unsigned long long sx, sy;  // elements between series (len * ld)
  int rows, cols, dim, ld;    // ld: row stride of the increments (inc_ld)
};

struct Outputs {
  double* d_values;              // indexed by output slot
  unsigned long long* d_err;     // indexed by output slot
  unsigned long long* d_maxrho;  // may be null
  double* d_grid;                // may be null
  double* d_diag;                // may be null
  unsigned long long grid_stride, diag_stride;
  unsigned long long* d_maxrho_all = nullptr;  // only the launch-wide max|rho| is wanted (SweepParams)
};

double flops_per_tile(int order, int dim) {
  const double n = order + 1;
  return 4.0 * n * n + 2.0 * dim;  // F(N, d)
}

int record_start(Ctx& c, StatRec* rec, sk_status* st) {
  if (!c.stats_on) return SK_OK;
  SK_CUDA(cudaEventCreate(&rec->a));
  SK_CUDA(cudaEventCreate(&rec->b));
  SK_CUDA(cudaEventRecord(rec->a, c.stream()));
  return SK_OK;
}

int record_end(Ctx& c, StatRec* rec, sk_status* st) {
  if (!c.stats_on) return SK_OK;
  SK_CUDA(cudaEventRecord(rec->b, c.stream()));
  c.stats.push_back(*rec);
  return SK_OK;
}

// Dependency-wait watchdog (SK_WATCHDOG_S, default 60 s): a sweep whose
// inter-band wait exceeds it aborts and reports instead of hanging the GPU.
unsigned long long watchdog_ns() {
  static const unsigned long long ns = [] {
    const char* e = std::getenv("SK_WATCHDOG_S");
    const double s = e ? std::atof(e) : 60.0;
    return static_cast<unsigned long long>((s > 0 ? s : 60.0) * 1e9);
  }();
  return ns;
}

// Host -> device copy of caller input on the context's stream.  A pageable
// buffer is copied through pinned staging by kStageWorkers host threads (4 MB
// chunks, two buffers each so a chunk's memcpy overlaps the previous chunk's
// DMA): 134 MB in 3.3 ms instead of 12.1 ms for a pageable cudaMemcpy on the
// B200 box (tools/h2d_staged_probe.cu).  Pinned or small inputs go straight.
constexpr int kStageWorkers = 8;
constexpr size_t kStageChunk = size_t(4) << 20;

cudaError_t h2d(Ctx& c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  bool pageable = bytes >= 4 * kStageChunk && std::getenv("SK_NO_STAGING") == nullptr;
  if (pageable) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, src) != cudaSuccess) {
      cudaGetLastError();
    } else if (a.type != cudaMemoryTypeUnregistered) {
      pageable = false;
    }
  }
  if (!pageable) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.stream());
  if (c.stage.empty()) {
    for (int k = 0; k < 2 * kStageWorkers; ++k) {
      void* p = nullptr;
      cudaEvent_t e = nullptr;
      if (cudaError_t err = cudaMallocHost(&p, kStageChunk); err != cudaSuccess) return err;
      c.stage.push_back(p);
      if (cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming); err != cudaSuccess) return err;
      c.stage_ev.push_back(e);
    }
    for (cudaEvent_t e : c.stage_ev) cudaEventRecord(e, c.stream());
  }
  const size_t nchunks = (bytes + kStageChunk - 1) / kStageChunk;
  const int device = c.device;
  cudaStream_t stream = c.stream();
  std::vector<cudaError_t> errs(kStageWorkers, cudaSuccess);
  std::vector<std::thread> th;
  for (int t = 0; t < kStageWorkers; ++t)
    th.emplace_back([&, t] {
      cudaSetDevice(device);
      int k = 0;
      for (size_t ch = t; ch < nchunks && errs[t] == cudaSuccess; ch += kStageWorkers, ++k) {
        const int b = 2 * t + (k & 1);
        // the DMA that last read this staging buffer has finished
        if ((errs[t] = cudaEventSynchronize(c.stage_ev[b])) != cudaSuccess) break;
        const size_t off = ch * kStageChunk, len = std::min(kStageChunk, bytes - off);
        std::memcpy(c.stage[b], static_cast<const char*>(src) + off, len);
        if ((errs[t] = cudaMemcpyAsync(static_cast<char*>(dst) + off, c.stage[b], len, cudaMemcpyHostToDevice,
                                       stream)) != cudaSuccess)
          break;
        errs[t] = cudaEventRecord(c.stage_ev[b], stream);
      }
    });
  for (auto& x : th) x.join();
  for (cudaError_t e : errs)
    if (e != cudaSuccess) return e;
  return cudaSuccess;
}

int check_watchdog(Ctx& c, sk_status* st) {
  unsigned long long h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  SK_CUDA(cudaMemcpyAsync(h, c.wd.p, sizeof h, cudaMemcpyDeviceToHost, c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
#ifdef SK_PROFILE_WAITS
  std::fprintf(stderr, "[sk] dependency waits: %.2f%% of band time (%.2f%% at band start)\n",
               h[7] ? 100.0 * h[6] / h[7] : 0.0, h[7] ? 100.0 * h[5] / h[7] : 0.0);
#endif
#ifdef SK_RHO_PROFILE
  std::fprintf(stderr, "[sk] rho ring: consumer waited %.3f ms, producer waited %.3f ms, producer busy %.3f ms (summed over bands)\n",
               h[5] * 1e-6, h[6] * 1e-6, h[7] * 1e-6);
#endif
  if (h[0] == 0) return SK_OK;
  return set_status(st, SK_INTERNAL, 0, 0,
                    "sweep watchdog: dependency wait timed out (pair %llu band %llu needs %llu, saw %llu)", h[1], h[2],
                    h[3], h[4]);
}

// Long pair over several GPUs (SweepParams::xgpus ...): this GPU's share of
// the block-cyclic band layout and the exchange areas of its block
// boundaries.  Default: every band, one GPU, no hand-off.
struct Strip {
  int gpus = 1, rank = 0, block = 0;  // block = 0: all bands in one block
  bool exch = false;
  bool emul = false;  // one launch over all `gpus` virtual GPUs (sk_propagate_split)
  const double* xin_abuf = nullptr;
  const unsigned long long* xin_prog = nullptr;
  double* xout_abuf = nullptr;
  unsigned long long* xout_prog = nullptr;
};

// Block-cyclic strip plan: blocks k = 0 .. nblocks-1 of `block` bands; GPU g
// owns k = g, g + G, ... (round r = k / G).  Returns the bands and rounds
// (column buffers) GPU `rank` sweeps and the exchange rounds it receives
// (blocks k >= 1 it owns: their bottom band's alpha comes from GPU k - 1).
struct StripPlan {
  size_t owned_bands = 0, rounds = 0, in_rounds = 0;
};
StripPlan strip_plan(size_t bands, size_t gpus, size_t rank, size_t block) {
  StripPlan pl;
  const size_t nblocks = (bands + block - 1) / block;
  for (size_t k = rank; k < nblocks; k += gpus) {
    pl.owned_bands += std::min(block, bands - k * block);
    pl.rounds = k / gpus + 1;
    if (k >= 1) pl.in_rounds = k / gpus + 1;
  }
  return pl;
}

// One persistent sweep launch per (order, pair chunk).  px/py/pout are
// launch-local pair lists of equal length.
int run_sweeps(Ctx& c, const PairSet& ps, const std::vector<uint32_t>& px, const std::vector<uint32_t>& py,
               const std::vector<uint32_t>& pout, int order, uint32_t flags, const Outputs& o, sk_status* st,
               const Strip& strip = Strip{}) {
  const size_t npairs_all = px.size();
  if (npairs_all == 0) return SK_OK;
  // test hook: every sweep with the reference's literal arithmetic
  if (const char* e = std::getenv("SK_FORCE_LITERAL"); e && e[0] == '1') flags |= kFlagLiteral | kFlagAllTotals;
  // literal re-sweeps run the register-resident literal kernel where it is
  // instantiated (order 8), the runtime-order literal kernel otherwise
  const bool lit = (flags & kFlagLiteral) && order == 8 && std::getenv("SK_NO_LIT_REG") == nullptr;
  const int ntempl = order <= kMaxRegOrder && (!(flags & kFlagLiteral) || lit) ? order : 0;
  const int dp = pick_dp(ps.dim);
  const int na = ntempl > 0 ? ntempl + 1 : kMaxOrder + 1;
  const int np = (na + 1) & ~1;
  const int rows = ps.rows, cols = ps.cols;
  const int band_rows = 32 * rows_per_lane(ntempl);  // 64-row bands for the register kernels
  const int bands = (rows + band_rows - 1) / band_rows;
  int bps = 0;
  const bool exact = o.d_maxrho != nullptr || lit;
  const bool extras = o.d_grid != nullptr || o.d_diag != nullptr || lit;
  const int okey = (((ntempl * 32 + dp) * 2 + (exact ? 1 : 0)) * 2 + (extras ? 1 : 0)) * 2 + (lit ? 1 : 0);
  if (auto it = c.occupancy.find(okey); it != c.occupancy.end()) {
    bps = it->second;
  } else {
    SK_CUDA(sweep_occupancy(ntempl, dp, exact, extras, lit, &bps));
    c.occupancy[okey] = bps;
  }
  if (bps < 1) return set_status(st, SK_CUDA_ERROR, 0, 0, "sweep kernel cannot be resident (occupancy 0)");
  Tracer tr;
  // free device memory for the workspace budgets below, refreshed every 32
  // launches (a heuristic input; allocation failures still surface)
  if (c.free_cache == 0 || ++c.free_age > 32) {
    size_t total_b = 0;
    SK_CUDA(cudaMemGetInfo(&c.free_cache, &total_b));
    c.free_age = 0;
  }
  const size_t free_b = c.free_cache;
  tr.mark("  occupancy+memgetinfo");
  // EXACT register kernels form the fast (fused) dot per tile and the
  // sequential one only where it could raise the exact max: they need a bound
  // on |fused - sequential| <= 2 d u sum|x_c y_c| <= 2 d u max||dx|| max||dy||
  double dot_err = 0.0;
  if (exact && ntempl > 0 && !lit) {
    const uint32_t nx = 1 + *std::max_element(px.begin(), px.end());
    const uint32_t ny = 1 + *std::max_element(py.begin(), py.end());
    SK_CUDA(c.sqn.ensure((nx + ny) * sizeof(double)));
    SK_CUDA(launch_max_sqnorm(ps.d_xinc, nx, cols, ps.dim, ps.ld, c.sqn.as<double>(), c.stream()));
    SK_CUDA(launch_max_sqnorm(ps.d_yinc, ny, rows, ps.dim, ps.ld, c.sqn.as<double>() + nx, c.stream()));
    c.aux_launches += 2;
    std::vector<double> h(nx + ny);
    SK_CUDA(cudaMemcpyAsync(h.data(), c.sqn.p, (nx + ny) * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
    SK_CUDA(cudaStreamSynchronize(c.stream()));
    const double mxx = *std::max_element(h.begin(), h.begin() + nx);
    const double mxy = *std::max_element(h.begin() + nx, h.end());
    dot_err = 4.0 * ps.dim * std::ldexp(1.0, -53) * std::sqrt(mxx * mxy) * 1.01 + 1e-300;
  }

  // Large d: a rho table per pair (rows x cols, one DMMA GEMM launch) when
  // the tables of a launch fit a quarter of the free memory (at most 8 GB),
  // else the band CTAs' producer warps form rho in shared memory -- O(l (N+d))
  // memory whatever the length.  Measured on cfg 4 (l = 16384, d = 512): GEMM
  // 8.7 ms + table sweep 19 ms vs fused 62 ms (the producers' L2 operand
  // traffic, ~0.5 MB per band per 32 columns, slows the bands' hand-off
  // chain), so the table wins where it fits.  SK_RHO_FUSED=1 forces fusion.
  const size_t tab_elems = dp == 0 ? static_cast<size_t>(rows) * cols : 0;
  const size_t tab_budget = std::min<size_t>(free_b / 4, size_t(8) << 30);
  const bool force_fused = std::getenv("SK_RHO_FUSED") != nullptr && std::getenv("SK_RHO_FUSED")[0] == '1';
  const bool use_table = dp == 0 && !force_fused && tab_elems * sizeof(double) <= tab_budget;
  size_t chunk = npairs_all;
  if (use_table) chunk = std::max<size_t>(1, tab_budget / (tab_elems * sizeof(double)));
  // units per launch must fit 32 bits
  chunk = std::min<size_t>(chunk, std::max<size_t>(1, (size_t(1) << 31) / bands));

  // Segment-DAG geometry (SweepParams::seg_cols).  The DAG of a pair is a
  // bands x segments grid worked in anti-diagonal waves: it needs enough units
  // per wave to fill the warps (pairs in flight x min(bands, segments)) and a
  // critical path ((bands + segments) x L steps) well below the per-warp
  // work.  The largest segment length L in {256, 128, 64} that meets both
  // (critical path under half the work, else under the work) is used;
  // otherwise the streaming schedule (a latency-bound short pair, multi-GPU
  // strips).
  const bool whole = strip.gpus == 1 && !strip.exch;
  const size_t sblock = strip.block > 0 ? static_cast<size_t>(strip.block) : static_cast<size_t>(bands);
  StripPlan plan = strip_plan(static_cast<size_t>(bands), static_cast<size_t>(strip.gpus),
                              static_cast<size_t>(strip.rank), sblock);
  const size_t xrounds = (((bands + sblock - 1) / sblock) + strip.gpus - 1) / strip.gpus;
  if (strip.emul) {
    plan.owned_bands = static_cast<size_t>(bands);
    plan.rounds = static_cast<size_t>(strip.gpus) * xrounds;
  }
  int seg_cols = 0;
  unsigned spb = 0, units_pair = 0;
  if (bands > 1 && whole && std::getenv("SK_STREAM") == nullptr) {
    const double warps_est = static_cast<double>(bps) * c.sms * band_workers(ntempl, dp);
    const double pairs_launch = static_cast<double>(std::min(chunk, npairs_all));
    const double active = std::min(pairs_launch, 2.0 * warps_est);
    const double work_steps = pairs_launch * bands * (cols + 31.0) / warps_est;
    const bool force = std::getenv("SK_FORCE_SEGMENTS") != nullptr;
    // measured (N = 8): 256 pairs x 4096^2 best at L = 256/128; one pair of
    // 262144^2 best at 64 (57 % vs 47 % streaming).  One pair alone: the
    // largest L whose waves still hold a unit per warp and whose critical
    // path fits in the work -- 10^6^2: L = 512, 13.97 s vs 15.2-15.6 s at 128
    // (256: 17.5, 1024: 17.2; two runs each, round 2)
    if (pairs_launch == 1.0 && !force) {
      for (int L : {512, 256, 128, 64}) {
        const double S = std::ceil((cols + 31.0) / L);
        if (std::min<double>(bands, S) >= warps_est && (bands + S) * L <= work_steps) {
          seg_cols = L;
          break;
        }
      }
    }
    for (const double crit_frac : {0.5, 1.0}) {
      if (seg_cols) break;
      for (int L : {256, 128, 64}) {
        const double S = std::ceil((cols + 31.0) / L);
        if (force ||
            (active * std::min<double>(bands, S) >= 2.0 * warps_est && (bands + S) * L <= crit_frac * work_steps)) {
          seg_cols = L;
          break;
        }
      }
      if (seg_cols) break;
    }
    if (const char* e = std::getenv("SK_SEG_COLS")) seg_cols = std::atoi(e);
  }
  if (seg_cols > 0) {
    seg_cols = std::max(band_rows, (seg_cols + band_rows - 1) / band_rows * band_rows);  // multiple of K and H
    for (int b = 0; b < bands; ++b) {
      const SegRange r = seg_range(rows, cols, b, band_rows, seg_cols);
      spb = std::max<unsigned>(spb, static_cast<unsigned>(r.hi - r.lo + 1));
      units_pair += static_cast<unsigned>(r.hi - r.lo + 1);
    }
    // the ready list holds every unit of a launch: at most 2^26 (256 MB)
    if (units_pair > (1u << 26)) seg_cols = 0;
    else chunk = std::min<size_t>(chunk, std::max<size_t>(1, (size_t(1) << 26) / units_pair));
    chunk = std::min<size_t>(chunk, std::max<size_t>(1, (size_t(1) << 31) / (static_cast<size_t>(bands) * spb)));
  }

  for (size_t c0 = 0; c0 < npairs_all; c0 += chunk) {
    const size_t npairs = std::min(chunk, npairs_all - c0);
    const int nb = static_cast<int>(plan.owned_bands);
    const unsigned long long units = static_cast<unsigned long long>(npairs) * nb;
    int blocks = bps * c.sms;
    if (const char* e = std::getenv("SK_FORCE_BPS")) blocks = std::max(1, std::min(bps, std::atoi(e))) * c.sms;
    const int per_block = band_workers(ntempl, dp);  // bands swept concurrently per CTA
    const unsigned long long need_blocks = (units + per_block - 1) / per_block;
    if (static_cast<unsigned long long>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
    const size_t warps = static_cast<size_t>(blocks) * per_block;
    size_t group = npairs >= warps ? warps : npairs;
    size_t slots = std::min(npairs, 2 * group);
    const size_t col_bytes = static_cast<size_t>(cols) * np * sizeof(double);
    if (bands > 1) {
      const size_t budget = std::max<size_t>(free_b / 4, col_bytes);
      const size_t fit = std::max<size_t>(1, budget / col_bytes);
      if (slots > fit) slots = std::max<size_t>(fit, 1);
      if (group > slots) group = slots;
    }
    // strips (one pair): one column buffer per block round
    if (!whole) {
      slots = plan.rounds;
      group = 1;
    }
    // test hooks: force small groups / slot counts to exercise slot reuse
    if (const char* e = std::getenv("SK_FORCE_GROUP")) group = std::max<size_t>(1, std::min<size_t>(group, std::atoi(e)));
    if (const char* e = std::getenv("SK_FORCE_SLOTS"))
      slots = std::max<size_t>(group, std::min<size_t>(slots, std::atoi(e)));
    // workspace
    SK_CUDA(c.pairs.ensure(3 * npairs * sizeof(uint32_t)));
    uint32_t* d_px = c.pairs.as<uint32_t>();
    uint32_t* d_py = d_px + npairs;
    uint32_t* d_po = d_py + npairs;
    SK_CUDA(cudaMemcpyAsync(d_px, px.data() + c0, npairs * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
    SK_CUDA(cudaMemcpyAsync(d_py, py.data() + c0, npairs * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
    SK_CUDA(cudaMemcpyAsync(d_po, pout.data() + c0, npairs * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
    SK_CUDA(c.prog.ensure(slots * bands * sizeof(unsigned long long)));
    SK_CUDA(cudaMemsetAsync(c.prog.p, 0, slots * bands * sizeof(unsigned long long), c.stream()));
    // [0] static unit order; SweepParams::ctr at +kCtrLine (one 128-byte line per counter)
    SK_CUDA(c.queue.ensure(4 * kCtrLine * sizeof(unsigned)));
    SK_CUDA(cudaMemsetAsync(c.queue.p, 0, 4 * kCtrLine * sizeof(unsigned), c.stream()));
    SK_CUDA(c.wd.ensure(8 * sizeof(unsigned long long)));
    SK_CUDA(cudaMemsetAsync(c.wd.p, 0, 8 * sizeof(unsigned long long), c.stream()));
    if (bands > 1) SK_CUDA(c.abuf.ensure(slots * col_bytes));
    // the DAG's lane-state records (slots x bands x ~5 KB) must fit next to
    // the column buffers; otherwise this launch streams
    const size_t rec_bytes = slots * static_cast<size_t>(bands) * susp_record_doubles(ntempl) * sizeof(double);
    const int seg_here = seg_cols > 0 && rec_bytes <= free_b / 4 ? seg_cols : 0;
    if (seg_here > 0) {
      const size_t nrec = slots * static_cast<size_t>(bands);
      SK_CUDA(c.susp.ensure(nrec * static_cast<size_t>(susp_record_doubles(ntempl)) * sizeof(double)));
      SK_CUDA(c.dep.ensure(nrec * spb * sizeof(unsigned)));
      SK_CUDA(cudaMemsetAsync(c.dep.p, 0, nrec * spb * sizeof(unsigned), c.stream()));
      const size_t ncell = npairs * static_cast<size_t>(units_pair);
      SK_CUDA(c.rq.ensure(ncell * sizeof(unsigned)));
      SK_CUDA(cudaMemsetAsync(c.rq.p, 0, ncell * sizeof(unsigned), c.stream()));
      // the first unit of each slot's first pair is ready
      const unsigned first = static_cast<unsigned>(std::min(slots, npairs));
      std::vector<unsigned> init(first + 1);
      for (unsigned k = 0; k < first; ++k) init[k] = k * static_cast<unsigned>(bands) * spb + 1u;
      SK_CUDA(cudaMemcpyAsync(c.rq.p, init.data(), first * sizeof(unsigned), cudaMemcpyHostToDevice, c.stream()));
      init[first] = first;
      SK_CUDA(cudaMemcpyAsync(c.queue.as<unsigned>() + 2 * kCtrLine, &init[first], sizeof(unsigned),
                              cudaMemcpyHostToDevice, c.stream()));
      SK_CUDA(cudaStreamSynchronize(c.stream()));  // `init` is pageable host memory
    }
    // cfg 4 (one large-d pair at a time, latency-bound sweep): the DMMA GEMM
    // runs beside the sweep on a second stream and publishes each 64-row
    // block as it completes; the sweep (compact layout, no producer warps)
    // leaves the SMs' tensor pipe, most issue slots and 110 KB of shared
    // memory free for it
    const bool overlap = use_table && ntempl > 0 && !lit && seg_here == 0 && group == 1 && whole &&
                         std::getenv("SK_NO_OVERLAP") == nullptr && c.ensure_side() == 0;
    const int nrb = (rows + 63) / 64, ncb = (cols + 63) / 64;
    if (use_table) {
      SK_CUDA(c.tab.ensure(npairs * tab_elems * sizeof(double)));
      if (overlap) {
        SK_CUDA(c.rowdone.ensure(npairs * nrb * sizeof(unsigned)));
        SK_CUDA(cudaMemsetAsync(c.rowdone.p, 0, npairs * nrb * sizeof(unsigned), c.stream()));
      } else {
        // exact (sequential) deltas for the literal kernel, DMMA otherwise (the
        // EXACT max|rho| re-forms candidates with the sequential dot)
        SK_CUDA(launch_rho_table(ps.d_xinc, ps.d_yinc, d_px, d_py, npairs, ps.sx, ps.sy, rows, cols, ps.dim, ps.ld,
                                 ntempl == 0 || lit, c.tab.as<double>(), tab_elems, c.stream()));
        ++c.aux_launches;
      }
    }
    SweepParams P{};
    P.xinc = ps.d_xinc;
    P.yinc = ps.d_yinc;
    P.pair_x = d_px;
    P.pair_y = d_py;
    P.pair_out = d_po;
    P.sx = ps.sx;
    P.sy = ps.sy;
    P.w65 = c.w65.as<double>() + ((flags & SK_W_FAULT) ? (kMaxOrder + 1) * (kMaxOrder + 1) : 0);
    P.dim = ps.dim;
    P.ld = ps.ld;
    P.rho_tab = use_table ? c.tab.as<double>() : nullptr;
    P.tab_stride = tab_elems;
    P.order = order;
    P.rows = rows;
    P.cols = cols;
    P.bands = bands;
    P.npairs = static_cast<int>(npairs);
    P.group = static_cast<int>(group);
    P.slots = static_cast<int>(slots);
    P.flags = flags;
    if (const char* e = std::getenv("SK_ALL_TOTALS"); e && e[0] == '1') P.flags |= kFlagAllTotals;
    P.abuf = bands > 1 ? c.abuf.as<double>() : nullptr;
    P.prog = c.prog.as<unsigned long long>();
    P.queue = c.queue.as<unsigned>();
    P.watchdog = c.wd.as<unsigned long long>();
    P.watchdog_ns = watchdog_ns();
    // with fewer pairs than warps, ~warps/group bands of each pair run at
    // once; when that is fewer than the pair's bands, a warp sweeps several
    // of them in turn and their natural spacing is one band time / (warps /
    // group).  With a warp per band the chain's hand-over is the only lag.
    P.start_lag = group < warps && warps < group * static_cast<size_t>(bands)
                      ? static_cast<int>(0.75 * (cols + 32.0) * group / warps)
                      : 0;
    P.dot_err = dot_err;
    if (const char* e = std::getenv("SK_START_LAG")) P.start_lag = std::atoi(e);
    // large d, table mode, one pair at a time, streaming, one GPU's whole
    // pair: consecutive bands share a CTA and hand alpha over in shared memory
    P.intra = dp == 0 && use_table && ntempl > 0 && seg_here == 0 && group == 1 && whole &&
              std::getenv("SK_NO_INTRA") == nullptr;
    P.values = o.d_values;
    P.err = o.d_err;
    P.maxrho = o.d_maxrho;
    P.maxrho_all = o.d_maxrho_all;
    P.grid = o.d_grid;
    P.diag = o.d_diag;
    P.grid_stride = o.grid_stride;
    P.diag_stride = o.diag_stride;
    P.xgpus = strip.gpus;
    P.xrank = strip.rank;
    P.xblock = static_cast<int>(sblock);
    P.xexch = strip.exch ? 1 : 0;
    P.xemul = strip.emul ? 1 : 0;
    P.xrounds = static_cast<int>(xrounds);
    P.units_pair_streaming = nb;
    P.xin_abuf = strip.xin_abuf;
    P.xin_prog = strip.xin_prog;
    P.xout_abuf = strip.xout_abuf;
    P.xout_prog = strip.xout_prog;
    P.seg_cols = seg_here;
    P.segs_per_band = static_cast<int>(spb);
    P.units_total = static_cast<unsigned>(npairs) * units_pair;
    P.susp = seg_here ? c.susp.as<double>() : nullptr;
    P.dep = seg_here ? c.dep.as<unsigned>() : nullptr;
    P.rq = seg_here ? c.rq.as<unsigned>() : nullptr;
    P.ctr = c.queue.as<unsigned>() + kCtrLine;

    if (overlap) {
      P.rho_ready = c.rowdone.as<unsigned>();
      P.rho_ready_need = static_cast<unsigned>(ncb);
      P.rho_ready_nrb = nrb;
      P.slot_stride = table_slot_doubles(ntempl);
    }

    StatRec rec{};
    rec.tiles = static_cast<double>(npairs) * rows * cols;
    rec.flops = rec.tiles * flops_per_tile(order, ps.dim);
    if (int rc = record_start(c, &rec, st)) return rc;
    if (overlap) {
      // the GEMM is queued FIRST: the sweep waits on it, never the reverse,
      // so even streams that the driver serialises (one hardware queue)
      // cannot deadlock -- they only lose the overlap
      SK_CUDA(cudaEventRecord(c.ev_fork, c.stream()));
      SK_CUDA(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
      SK_CUDA(launch_rho_table(ps.d_xinc, ps.d_yinc, d_px, d_py, npairs, ps.sx, ps.sy, rows, cols, ps.dim, ps.ld,
                               false, c.tab.as<double>(), tab_elems, c.side, c.rowdone.as<unsigned>()));
      ++c.aux_launches;
    }
    SK_CUDA(sweep_launch(ntempl, dp, exact, extras, lit, blocks, c.stream(), P));
    if (overlap) {
      SK_CUDA(cudaEventRecord(c.ev_join, c.side));
      SK_CUDA(cudaStreamWaitEvent(c.stream(), c.ev_join, 0));
    }
    if (int rc = record_end(c, &rec, st)) return rc;
    ++c.sweep_launches;
    if (int rc = check_watchdog(c, st)) return rc;
  }
  return SK_OK;
}

// Per-pair truncation order (wavefront.cpp:206-221 / gram.cpp:57-64).
// estimate_order is monotone in max|rho| and never below 8, so when the
// Cauchy-Schwarz bound U >= max|rho| already yields N = 8 that is the exact
// answer; only the other pairs pay for the O(l^2 d) exact scan.
int adaptive_orders(Ctx& c, const PairSet& ps, const std::vector<double>& h_sqn_x,
                    const std::vector<double>& h_sqn_y, const std::vector<uint32_t>& px,
                    const std::vector<uint32_t>& py, double tol, std::vector<int>& orders, std::vector<int>& conv,
                    sk_status* st) {
  const size_t np = px.size();
  orders.assign(np, 8);
  conv.assign(np, 1);
  const double slack = 1e-10 + 8.0 * (ps.dim + 2) * std::ldexp(1.0, -53);
  std::vector<uint32_t> sx_list, sy_list, idx;
  for (size_t k = 0; k < np; ++k) {
    const double u = std::sqrt(h_sqn_x[px[k]]) * std::sqrt(h_sqn_y[py[k]]) * (1.0 + slack);
    int ord = 0, cv = 0;
    if (std::isfinite(u)) host_estimate_order(u, tol, &ord, &cv);
    if (std::isfinite(u) && ord == 8 && cv) continue;
    sx_list.push_back(px[k]);
    sy_list.push_back(py[k]);
    idx.push_back(static_cast<uint32_t>(k));
  }
  if (idx.empty()) return SK_OK;
  const size_t ns = idx.size();
  SK_CUDA(c.pairs.ensure(2 * ns * sizeof(uint32_t)));
  SK_CUDA(c.scan.ensure(ns * sizeof(unsigned long long)));
  uint32_t* d_px = c.pairs.as<uint32_t>();
  uint32_t* d_py = d_px + ns;
  SK_CUDA(cudaMemcpyAsync(d_px, sx_list.data(), ns * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
  SK_CUDA(cudaMemcpyAsync(d_py, sy_list.data(), ns * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
  SK_CUDA(cudaMemsetAsync(c.scan.p, 0, ns * sizeof(unsigned long long), c.stream()));
  SK_CUDA(launch_maxrho_scan(ps.d_xinc, ps.d_yinc, d_px, d_py, ns, ps.sx, ps.sy, ps.rows, ps.cols, ps.dim, ps.ld,
                             c.scan.as<unsigned long long>(), c.stream()));
  ++c.aux_launches;
  std::vector<unsigned long long> bits(ns);
  SK_CUDA(cudaMemcpyAsync(bits.data(), c.scan.p, ns * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  for (size_t t = 0; t < ns; ++t) {
    double mr;
    std::memcpy(&mr, &bits[t], sizeof mr);
    if (mr < 0.0 || !std::isfinite(mr))
      return set_status(st, SK_INVALID_ARGUMENT, 0, 0,
                        "estimate_order: max_abs_rho must be finite and nonnegative");
    host_estimate_order(mr, tol, &orders[idx[t]], &conv[idx[t]]);
  }
  return SK_OK;
}

// decode an error key into the reference's exception contract; `delta` is the
// failing tile's increment product for the overflow message (NaN if unknown)
int decode_err(unsigned long long key, sk_status* st, double delta) {
  const unsigned code = static_cast<unsigned>(key & 3ull);
  const uint64_t i = (key >> 2) & 0x3fffffffull;
  const uint64_t d = key >> 32;
  const uint64_t j = d - i;
  if (code == kErrDelta)
    return set_status(st, SK_NUMERIC_OVERFLOW, j + 1, i + 1,
                      "increment product %f on tile (%llu, %llu) exceeds double range at any order; rescale "
                      "the inputs",
                      delta, static_cast<unsigned long long>(j + 1), static_cast<unsigned long long>(i + 1));
  if (code == kErrCorner)
    return set_status(st, SK_INCONSISTENT_BOUNDARY, j + 1, i + 1,
                      "boundary series disagree at the shared corner on tile (%llu, %llu)",
                      static_cast<unsigned long long>(j + 1), static_cast<unsigned long long>(i + 1));
  return set_status(st, SK_NUMERIC_OVERFLOW, j + 1, i + 1,
                    "non-finite series on tile (%llu, %llu); rescale the inputs or reduce the order",
                    static_cast<unsigned long long>(j + 1), static_cast<unsigned long long>(i + 1));
}

// The failing tile's increment product for the overflow message
// (wavefront.cpp:146-155): the two increment rows (device layout: row k + 1
// holds dz_k, stride ld) come back and are dotted in the reference's order.
// xs / ys: device increments of the pair's x and y series.  NaN unless `key`
// is an increment-product overflow.
double device_delta(Ctx& c, const double* xs, const double* ys, size_t ld, size_t dim, unsigned long long key) {
  if ((key & 3ull) != kErrDelta) return std::numeric_limits<double>::quiet_NaN();
  const uint64_t i = (key >> 2) & 0x3fffffffull;
  const uint64_t j = (key >> 32) - i;
  std::vector<double> a(ld), b(ld);
  if (cudaMemcpyAsync(a.data(), xs + (j + 1) * ld, ld * sizeof(double), cudaMemcpyDeviceToHost, c.stream()) !=
          cudaSuccess ||
      cudaMemcpyAsync(b.data(), ys + (i + 1) * ld, ld * sizeof(double), cudaMemcpyDeviceToHost, c.stream()) !=
          cudaSuccess ||
      cudaStreamSynchronize(c.stream()) != cudaSuccess) {
    cudaGetLastError();
    return std::numeric_limits<double>::quiet_NaN();
  }
  double acc = 0.0;
  for (size_t q = 0; q < dim; ++q) acc += a[q] * b[q];
  return acc;
}

// Second sweeps after a throughput launch (launch index t writes output slot
// t: values / err on the device, hv / he on the host).
//  * Strict corner screen: a register-kernel pair whose first flagged tile is
//    a corner screen (kCornerScreen, sk_device.cuh) is swept again with the
//    literal kernel, which repeats the reference bit for bit -- so the
//    reference's throw, its tile, or the value it returns, exactly.
//  * Partial totals: throughput sweeps form tile totals only where a pair's
//    final tile can fall (kFlagAllTotals).  A pair that ended flagged (its
//    first failure may be preceded by an unchecked non-finite tile) or
//    non-finite is swept again with every total formed and checked: the
//    reference's first failing tile, exactly.  Not needed when the first
//    sweep already formed every total (`all_totals`).
// The flagged slots are reset by one scatter kernel, re-swept, and read back
// with one gather (no per-pair API calls).
int recheck_failures(Ctx& c, const PairSet& ps, const std::vector<uint32_t>& px, const std::vector<uint32_t>& py,
                     const std::vector<int>& ords, uint32_t flags, const Outputs& o, std::vector<double>& hv,
                     std::vector<unsigned long long>& he, bool all_totals, sk_status* st) {
  std::vector<uint32_t> literal, totals;
  for (size_t t = 0; t < he.size(); ++t) {
    const bool corner = he[t] != ~0ull && (he[t] & 3ull) == kErrCorner;
    if (corner && ords[t] <= kMaxRegOrder && (flags & kFlagStrictCorner))
      literal.push_back(static_cast<uint32_t>(t));
    else if (!all_totals && (he[t] != ~0ull || !std::isfinite(hv[t])))
      totals.push_back(static_cast<uint32_t>(t));
  }
  if (literal.empty() && totals.empty()) return SK_OK;
  for (int pass = 0; pass < 2; ++pass) {
    const std::vector<uint32_t>& redo = pass == 0 ? literal : totals;
    if (redo.empty()) continue;
    const uint32_t extra = pass == 0 ? (kFlagLiteral | kFlagAllTotals) : kFlagAllTotals;
    SK_CUDA(c.redo.ensure(redo.size() * sizeof(uint32_t)));
    SK_CUDA(cudaMemcpyAsync(c.redo.p, redo.data(), redo.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                            c.stream()));
    SK_CUDA(launch_reset_slots(c.redo.as<uint32_t>(), redo.size(), o.d_err, c.stream()));
    ++c.aux_launches;
    std::vector<int> distinct;
    for (uint32_t t : redo) distinct.push_back(ords[t]);
    std::sort(distinct.begin(), distinct.end());
    distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
    for (int ord : distinct) {
      std::vector<uint32_t> gx, gy, go;
      for (uint32_t t : redo)
        if (ords[t] == ord) {
          gx.push_back(px[t]);
          gy.push_back(py[t]);
          go.push_back(t);
        }
      if (int rc = run_sweeps(c, ps, gx, gy, go, ord, flags | extra, o, st)) return rc;
      if (pass == 0) c.literal_rechecks += gx.size();
    }
    // one gather of the re-swept slots' values and error keys
    const size_t nr = redo.size();
    SK_CUDA(c.redo_out.ensure(nr * 2 * sizeof(unsigned long long)));
    SK_CUDA(launch_gather_slots(c.redo.as<uint32_t>(), nr, o.d_values, o.d_err,
                                c.redo_out.as<unsigned long long>(), c.stream()));
    ++c.aux_launches;
    std::vector<unsigned long long> back(2 * nr);
    SK_CUDA(cudaMemcpyAsync(back.data(), c.redo_out.p, back.size() * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c.stream()));
    SK_CUDA(cudaStreamSynchronize(c.stream()));
    for (size_t q = 0; q < nr; ++q) {
      std::memcpy(&hv[redo[q]], &back[q], sizeof(double));
      he[redo[q]] = back[nr + q];
    }
  }
  return SK_OK;
}

// Pairwise core on device-resident raw series.  values: device, npairs.
struct PairwiseResult {
  std::vector<int> orders, conv;
  std::vector<unsigned long long> err;
  std::vector<unsigned long long> maxr;
};

int pairwise_core(Ctx& c, const double* d_xraw, size_t lx, const double* d_yraw, size_t ly, size_t npairs,
                  size_t dim, int adaptive, int order, double tol, uint32_t flags, double* d_values,
                  bool want_maxrho, double* d_grid, double* d_diag, PairwiseResult& res, sk_status* st) {
  Tracer tr;
  const size_t cx = lx - 1, cy = ly - 1;
  const size_t ld = inc_ld(dim);
  SK_CUDA(c.xinc.ensure(npairs * lx * ld * sizeof(double)));
  SK_CUDA(c.yinc.ensure(npairs * ly * ld * sizeof(double)));
  // with the adaptive policy the per-series max squared increment norms come
  // out of the same pass (the order proof below)
  if (adaptive) SK_CUDA(c.sqn.ensure(2 * npairs * sizeof(double)));
  SK_CUDA(launch_increments(d_xraw, npairs, lx, dim, ld, c.xinc.as<double>(), c.stream(),
                            adaptive ? c.sqn.as<double>() : nullptr));
  SK_CUDA(launch_increments(d_yraw, npairs, ly, dim, ld, c.yinc.as<double>(), c.stream(),
                            adaptive ? c.sqn.as<double>() + npairs : nullptr));
  c.aux_launches += adaptive && ld > 16 ? 4 : 2;
  PairSet ps{c.xinc.as<double>(), c.yinc.as<double>(), lx * ld, ly * ld, static_cast<int>(cy),
             static_cast<int>(cx), static_cast<int>(dim), static_cast<int>(ld)};
  std::vector<uint32_t> px(npairs), py(npairs), pout(npairs);
  for (size_t k = 0; k < npairs; ++k) px[k] = py[k] = pout[k] = static_cast<uint32_t>(k);
  if (adaptive) {
    std::vector<double> h(2 * npairs);
    SK_CUDA(cudaMemcpyAsync(h.data(), c.sqn.p, 2 * npairs * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
    SK_CUDA(cudaStreamSynchronize(c.stream()));
    tr.mark("increments+norms (sync)");
    std::vector<double> hx(h.begin(), h.begin() + npairs), hy(h.begin() + npairs, h.end());
    if (int rc = adaptive_orders(c, ps, hx, hy, px, py, tol, res.orders, res.conv, st)) return rc;
    tr.mark("adaptive orders");
  } else {
    res.orders.assign(npairs, order);
    res.conv.assign(npairs, 1);
  }
  SK_CUDA(c.err.ensure(npairs * sizeof(unsigned long long)));
  SK_CUDA(cudaMemsetAsync(c.err.p, 0xff, npairs * sizeof(unsigned long long), c.stream()));
  SK_CUDA(cudaMemsetAsync(d_values, 0xff, npairs * sizeof(double), c.stream()));
  if (want_maxrho) {
    SK_CUDA(c.maxr.ensure(npairs * sizeof(unsigned long long)));
    SK_CUDA(cudaMemsetAsync(c.maxr.p, 0, npairs * sizeof(unsigned long long), c.stream()));
  }
  Outputs o{d_values, c.err.as<unsigned long long>(), want_maxrho ? c.maxr.as<unsigned long long>() : nullptr,
            d_grid, d_diag, lx * ly, std::min(cx, cy)};
  // one sweep per distinct order
  std::vector<int> distinct(res.orders.begin(), res.orders.end());
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  for (int ord : distinct) {
    std::vector<uint32_t> gx, gy, go;
    for (size_t k = 0; k < npairs; ++k)
      if (res.orders[k] == ord) {
        gx.push_back(px[k]);
        gy.push_back(py[k]);
        go.push_back(pout[k]);
      }
    if (int rc = run_sweeps(c, ps, gx, gy, go, ord, flags, o, st)) return rc;
  }
  tr.mark("sweep launch (async)");
  res.err.resize(npairs);
  std::vector<double> hv(npairs);
  SK_CUDA(cudaMemcpyAsync(res.err.data(), c.err.p, npairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c.stream()));
  SK_CUDA(cudaMemcpyAsync(hv.data(), d_values, npairs * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
  if (want_maxrho) {
    res.maxr.resize(npairs);
    SK_CUDA(cudaMemcpyAsync(res.maxr.data(), c.maxr.p, npairs * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c.stream()));
  }
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  SK_CUDA(cudaGetLastError());
  tr.mark("sweep done (sync)");
  // knot-grid sweeps form every total already (the diagonal only near tiles (i, i))
  if (int rc = recheck_failures(c, ps, px, py, res.orders, flags, o, hv, res.err, d_grid != nullptr, st)) return rc;
  return SK_OK;
}


int gram_validate(size_t m, size_t len, size_t dim, int adaptive, int order, double tol, sk_status* st) {
  if (m == 0) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "gram_matrix: family must be nonempty");
  if (dim < 1) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "gram_matrix: dimension must be >= 1");
  if (len < 2) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "gram_matrix: common length must be >= 2");
  if (adaptive ? !(tol > 0.0) : (order < 1 || order > kMaxOrder))
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, adaptive ? "adaptive tolerance must be positive"
                                                             : "propagate: order must lie in [1, 64]");
  return SK_OK;
}

// Gram core over device-resident raw series (family, m x len x dim): the
// upper-triangle pairs [t0, t1) in row-major order (gram.cpp:39-42), as
// gram.cpp:51-66 evaluates each entry -- increments, order (pre-pass proof or
// exact scan), one sweep per distinct order, re-sweeps.  Leaves per-pair
// results (launch slot t = pair t0 + t) on the host in `g` and the values /
// error keys on the device (c.values, c.err); the failure records of the call
// go to c.failures.
struct GramCore {
  std::vector<uint32_t> pi, pj;
  std::vector<int> ords, conv;
  std::vector<double> hv;
  std::vector<unsigned long long> he, hm;
};

int gram_core(Ctx& c, const double* d_family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
              uint32_t flags, bool want_max, bool per_pair_max, size_t t0, size_t t1, GramCore& g,
              sk_status* st) {
  c.failures.clear();
  const size_t np = t1 - t0;
  if (np == 0) return SK_OK;
  // upper-triangle pairs (i <= j), row-major: locate t0, then walk
  g.pi.resize(np);
  g.pj.resize(np);
  std::vector<uint32_t> pout(np);
  {
    size_t i = 0, row_start = 0;
    while (i < m && row_start + (m - i) <= t0) {
      row_start += m - i;
      ++i;
    }
    size_t j = i + (t0 - row_start);
    for (size_t t = 0; t < np; ++t) {
      g.pi[t] = static_cast<uint32_t>(i);
      g.pj[t] = static_cast<uint32_t>(j);
      pout[t] = static_cast<uint32_t>(t);
      if (++j == m) {
        ++i;
        j = i;
      }
    }
  }
  const size_t cnt = len - 1;
  const size_t ld = inc_ld(dim);
  SK_CUDA(c.xinc.ensure(m * len * ld * sizeof(double)));
  SK_CUDA(c.values.ensure(np * sizeof(double)));
  if (adaptive) SK_CUDA(c.sqn.ensure(m * sizeof(double)));
  SK_CUDA(launch_increments(d_family, m, len, dim, ld, c.xinc.as<double>(), c.stream(),
                            adaptive ? c.sqn.as<double>() : nullptr));
  c.aux_launches += adaptive && ld > 16 ? 2 : 1;
  // propagate(padded[i], padded[j]): x = member i (columns), y = member j (rows)
  PairSet ps{c.xinc.as<double>(), c.xinc.as<double>(), len * ld, len * ld, static_cast<int>(cnt),
             static_cast<int>(cnt), static_cast<int>(dim), static_cast<int>(ld)};
  if (adaptive) {
    std::vector<double> h(m);
    SK_CUDA(cudaMemcpyAsync(h.data(), c.sqn.p, m * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
    SK_CUDA(cudaStreamSynchronize(c.stream()));
    if (int rc = adaptive_orders(c, ps, h, h, g.pi, g.pj, tol, g.ords, g.conv, st)) return rc;
  } else {
    g.ords.assign(np, order);
    g.conv.assign(np, 1);
  }
  SK_CUDA(c.err.ensure(np * sizeof(unsigned long long)));
  SK_CUDA(cudaMemsetAsync(c.err.p, 0xff, np * sizeof(unsigned long long), c.stream()));
  SK_CUDA(cudaMemsetAsync(c.values.p, 0xff, np * sizeof(double), c.stream()));
  if (want_max) {
    SK_CUDA(c.maxr.ensure(np * sizeof(unsigned long long)));
    SK_CUDA(cudaMemsetAsync(c.maxr.p, 0, np * sizeof(unsigned long long), c.stream()));
  }
  Outputs o{c.values.as<double>(), c.err.as<unsigned long long>(),
            want_max ? c.maxr.as<unsigned long long>() : nullptr, nullptr, nullptr, 0, 0};
  if (want_max && !per_pair_max) {
    // only the family's maximum is reported: one running max for the launch
    SK_CUDA(c.maxall.ensure(sizeof(unsigned long long)));
    SK_CUDA(cudaMemsetAsync(c.maxall.p, 0, sizeof(unsigned long long), c.stream()));
    o.d_maxrho_all = c.maxall.as<unsigned long long>();
  }
  std::vector<int> distinct(g.ords.begin(), g.ords.end());
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  for (int ord : distinct) {
    std::vector<uint32_t> gx, gy, go;
    for (size_t k = 0; k < np; ++k)
      if (g.ords[k] == ord) {
        gx.push_back(g.pi[k]);
        gy.push_back(g.pj[k]);
        go.push_back(pout[k]);
      }
    if (int rc = run_sweeps(c, ps, gx, gy, go, ord, flags, o, st)) return rc;
  }
  g.hv.resize(np);
  g.he.resize(np);
  g.hm.assign(want_max ? np : 0, 0ull);
  SK_CUDA(cudaMemcpyAsync(g.hv.data(), c.values.p, np * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
  SK_CUDA(cudaMemcpyAsync(g.he.data(), c.err.p, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.stream()));
  if (want_max)
    SK_CUDA(cudaMemcpyAsync(g.hm.data(), c.maxr.p, np * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  SK_CUDA(cudaGetLastError());
  if (int rc = recheck_failures(c, ps, g.pi, g.pj, g.ords, flags, o, g.hv, g.he, false, st)) return rc;
  // gram.cpp:74-77: overflow entries become NaN + a failure record; anything
  // else (the corner check) aborts the call with the first such entry's error
  for (size_t t = 0; t < np; ++t) {
    if (g.he[t] == ~0ull) continue;
    if ((g.he[t] & 3ull) == kErrCorner) {
      const unsigned long long key = g.he[t];
      return decode_err(key, st, std::numeric_limits<double>::quiet_NaN());
    }
    sk_gram_failure f{};
    f.row = g.pi[t];
    f.col = g.pj[t];
    decode_err(g.he[t], &f.status,
               device_delta(c, ps.d_xinc + g.pi[t] * ps.sx, ps.d_xinc + g.pj[t] * ps.sx, ld, dim, g.he[t]));
    c.failures.push_back(f);
  }
  return SK_OK;
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int sk_abi_version(void) { return SK_ABI_VERSION; }

int sk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sk_set_device(int device, sk_status* st) {
  clear_status(st);
  const int n = sk_device_count();
  if (device < 0 || device >= n)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "device %d out of range (%d visible)", device, n);
  t_device = device;
  return SK_OK;
}

int sk_set_stream(void* cuda_stream, sk_status* st) {
  clear_status(st);
  Ctx* c = nullptr;
  if (int rc = get_ctx(&c, st)) return rc;
  c->user = static_cast<cudaStream_t>(cuda_stream);
  return SK_OK;
}

int sk_estimate_order(double max_abs_rho, size_t /*length*/, double tol, int* order, int* converged,
                      sk_status* st) {
  clear_status(st);
  if (!(tol > 0.0)) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "estimate_order: tolerance must be positive");
  if (max_abs_rho < 0.0 || !std::isfinite(max_abs_rho))
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "estimate_order: max_abs_rho must be finite and nonnegative");
  return host_estimate_order(max_abs_rho, tol, order, converged);
}

int sk_propagate(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order, uint32_t flags,
                 double* value, uint64_t* peak_live, double* grid, double* diag, sk_status* st) {
  clear_status(st);
  if (dim < 1) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate: series dimensions differ");
  if (lx < 2 || ly < 2) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate: both series need length >= 2");
  if (order < 1 || order > kMaxOrder)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate: order must lie in [1, 64]");
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  SK_CUDA(c.raw_x.ensure(lx * dim * sizeof(double)));
  SK_CUDA(c.raw_y.ensure(ly * dim * sizeof(double)));
  SK_CUDA(c.values.ensure(sizeof(double)));
  SK_CUDA(h2d(c, c.raw_x.p, x, lx * dim * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_y.p, y, ly * dim * sizeof(double)));
  double* d_grid = nullptr;
  double* d_diag = nullptr;
  if (grid) {
    SK_CUDA(c.grid.ensure(lx * ly * sizeof(double)));
    d_grid = c.grid.as<double>();
    SK_CUDA(cudaMemsetAsync(d_grid, 0, lx * ly * sizeof(double), c.stream()));
    SK_CUDA(launch_grid_init(d_grid, 1, lx, ly, c.stream()));
  }
  const size_t nd = std::min(lx, ly) - 1;
  if (diag) {
    SK_CUDA(c.diag.ensure(nd * sizeof(double)));
    d_diag = c.diag.as<double>();
  }
  PairwiseResult res;
  if (int rc = pairwise_core(c, c.raw_x.as<double>(), lx, c.raw_y.as<double>(), ly, 1, dim, 0, order, 1e-12, flags,
                             c.values.as<double>(), false, d_grid, d_diag, res, st))
    return rc;
  if (res.err[0] != ~0ull)
    return decode_err(res.err[0], st, device_delta(c, c.xinc.as<double>(), c.yinc.as<double>(), inc_ld(dim), dim,
                                                   res.err[0]));
  SK_CUDA(cudaMemcpy(value, c.values.p, sizeof(double), cudaMemcpyDeviceToHost));
  if (grid) SK_CUDA(cudaMemcpy(grid, d_grid, lx * ly * sizeof(double), cudaMemcpyDeviceToHost));
  if (diag) SK_CUDA(cudaMemcpy(diag, d_diag, nd * sizeof(double), cudaMemcpyDeviceToHost));
  if (peak_live) *peak_live = peak_live_closed_form(ly - 1, lx - 1);
  return SK_OK;
}

int sk_max_abs_rho(const double* x, size_t lx, const double* y, size_t ly, size_t dim, double* out, sk_status* st) {
  clear_status(st);
  if (dim < 1 || lx < 2 || ly < 2)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "increments: a single point has no increments");
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  SK_CUDA(c.raw_x.ensure(lx * dim * sizeof(double)));
  SK_CUDA(c.raw_y.ensure(ly * dim * sizeof(double)));
  const size_t ld = inc_ld(dim);
  SK_CUDA(c.xinc.ensure(lx * ld * sizeof(double)));
  SK_CUDA(c.yinc.ensure(ly * ld * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_x.p, x, lx * dim * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_y.p, y, ly * dim * sizeof(double)));
  SK_CUDA(launch_increments(c.raw_x.as<double>(), 1, lx, dim, ld, c.xinc.as<double>(), c.stream()));
  SK_CUDA(launch_increments(c.raw_y.as<double>(), 1, ly, dim, ld, c.yinc.as<double>(), c.stream()));
  SK_CUDA(c.pairs.ensure(2 * sizeof(uint32_t)));
  SK_CUDA(cudaMemsetAsync(c.pairs.p, 0, 2 * sizeof(uint32_t), c.stream()));
  SK_CUDA(c.scan.ensure(sizeof(unsigned long long)));
  SK_CUDA(cudaMemsetAsync(c.scan.p, 0, sizeof(unsigned long long), c.stream()));
  uint32_t* d_p = c.pairs.as<uint32_t>();
  SK_CUDA(launch_maxrho_scan(c.xinc.as<double>(), c.yinc.as<double>(), d_p, d_p + 1, 1, 0, 0,
                             static_cast<int>(ly - 1), static_cast<int>(lx - 1), static_cast<int>(dim),
                             static_cast<int>(ld), c.scan.as<unsigned long long>(), c.stream()));
  c.aux_launches += 3;
  unsigned long long bits = 0;
  SK_CUDA(cudaMemcpyAsync(&bits, c.scan.p, sizeof bits, cudaMemcpyDeviceToHost, c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  std::memcpy(out, &bits, sizeof(double));
  return SK_OK;
}

static int step_tile_common(bool fast, double delta, const double* alpha, const double* beta, int order,
                            double* out_alpha, double* out_beta, double* total, sk_status* st) {
  clear_status(st);
  if (order < 0 || order > kMaxOrder)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "step_tile: order must lie in [0, 64]");
  if (fast && (order < 1 || order > kMaxRegOrder))
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "step_tile_fast: order must lie in [1, 16]");
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  const int n = order + 1;
  std::vector<double> in(2 * (kMaxOrder + 1), 0.0), out(2 * (kMaxOrder + 1) + 1, 0.0);
  std::copy(alpha, alpha + n, in.begin());
  std::copy(beta, beta + n, in.begin() + (kMaxOrder + 1));
  SK_CUDA(c.tile_io.ensure((in.size() + out.size()) * sizeof(double)));
  double* d_in = c.tile_io.as<double>();
  double* d_out = d_in + in.size();
  SK_CUDA(cudaMemcpyAsync(d_in, in.data(), in.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream()));
  if (fast) {
    SK_CUDA(launch_step_tile_fast(delta, order, d_in, d_out, c.stream()));
  } else {
    SK_CUDA(launch_step_tile_literal(delta, order, c.w65.as<double>(), d_in, d_out, c.stream()));
  }
  ++c.aux_launches;
  SK_CUDA(cudaMemcpyAsync(out.data(), d_out, out.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  std::copy(out.begin(), out.begin() + n, out_alpha);
  std::copy(out.begin() + (kMaxOrder + 1), out.begin() + (kMaxOrder + 1) + n, out_beta);
  if (total) *total = out[2 * (kMaxOrder + 1)];
  return SK_OK;
}

int sk_step_tile(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                 double* out_beta, double* total, sk_status* st) {
  return step_tile_common(false, delta, alpha, beta, order, out_alpha, out_beta, total, st);
}

int sk_step_tile_fast(double delta, const double* alpha, const double* beta, int order, double* out_alpha,
                      double* out_beta, double* total, sk_status* st) {
  return step_tile_common(true, delta, alpha, beta, order, out_alpha, out_beta, total, st);
}

static int pairwise_validate(size_t lx, size_t ly, size_t dim, int adaptive, int order, double tol, sk_status* st) {
  if (dim < 1) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "pairwise: dimension must be >= 1");
  if (lx < 2 || ly < 2) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate: both series need length >= 2");
  if (adaptive) {
    if (!(tol > 0.0)) return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "adaptive tolerance must be positive");
  } else if (order < 1 || order > kMaxOrder) {
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate: order must lie in [1, 64]");
  }
  return SK_OK;
}

static void fill_pair_outputs(Ctx& c, const PairwiseResult& res, size_t npairs, double* values, int* orders,
                              int* converged, double* max_abs_rho, sk_status* per_pair, size_t lx, size_t ly,
                              size_t dim) {
  const size_t ld = inc_ld(dim);
  for (size_t k = 0; k < npairs; ++k) {
    if (orders) orders[k] = res.orders[k];
    if (converged) converged[k] = res.conv[k];
    if (max_abs_rho && !res.maxr.empty()) std::memcpy(&max_abs_rho[k], &res.maxr[k], sizeof(double));
    if (res.err[k] != ~0ull) {
      if (values) values[k] = std::numeric_limits<double>::quiet_NaN();
      if (per_pair)
        decode_err(res.err[k], &per_pair[k],
                   device_delta(c, c.xinc.as<double>() + k * lx * ld, c.yinc.as<double>() + k * ly * ld, ld, dim,
                                res.err[k]));
    } else if (per_pair) {
      clear_status(&per_pair[k]);
    }
  }
}

int sk_pairwise(const double* xs, size_t lx, const double* ys, size_t ly, size_t npairs, size_t dim, int adaptive,
                int order, double tol, uint32_t flags, double* values, int* orders, int* converged,
                double* max_abs_rho, sk_status* per_pair, sk_status* st) {
  clear_status(st);
  if (npairs == 0) return SK_OK;
  if (int rc = pairwise_validate(lx, ly, dim, adaptive, order, tol, st)) return rc;
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  SK_CUDA(c.raw_x.ensure(npairs * lx * dim * sizeof(double)));
  SK_CUDA(c.raw_y.ensure(npairs * ly * dim * sizeof(double)));
  SK_CUDA(c.values.ensure(npairs * sizeof(double)));
  Tracer tr;
  SK_CUDA(h2d(c, c.raw_x.p, xs, npairs * lx * dim * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_y.p, ys, npairs * ly * dim * sizeof(double)));
  tr.mark("pairwise: h2d issued");
  PairwiseResult res;
  if (int rc = pairwise_core(c, c.raw_x.as<double>(), lx, c.raw_y.as<double>(), ly, npairs, dim, adaptive, order,
                             tol, flags, c.values.as<double>(), max_abs_rho != nullptr, nullptr, nullptr, res, st))
    return rc;
  tr.mark("pairwise: core");
  SK_CUDA(cudaMemcpy(values, c.values.p, npairs * sizeof(double), cudaMemcpyDeviceToHost));
  fill_pair_outputs(c, res, npairs, values, orders, converged, max_abs_rho, per_pair, lx, ly, dim);
  tr.mark("pairwise: outputs");
  return SK_OK;
}

int sk_pairwise_device(const double* d_xs, size_t lx, const double* d_ys, size_t ly, size_t npairs, size_t dim,
                       int adaptive, int order, double tol, uint32_t flags, double* d_values, int* orders,
                       int* converged, sk_status* per_pair, sk_status* st) {
  clear_status(st);
  if (npairs == 0) return SK_OK;
  if (int rc = pairwise_validate(lx, ly, dim, adaptive, order, tol, st)) return rc;
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  PairwiseResult res;
  if (int rc = pairwise_core(*cp, d_xs, lx, d_ys, ly, npairs, dim, adaptive, order, tol, flags, d_values, false,
                             nullptr, nullptr, res, st))
    return rc;
  fill_pair_outputs(*cp, res, npairs, nullptr, orders, converged, nullptr, per_pair, lx, ly, dim);
  return SK_OK;
}

int sk_gram(const double* family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
            uint32_t flags, int scan_products, size_t shard, size_t nshards, double* values, int* orders,
            double* pair_max, double* max_product, int* converged, size_t* n_failures, sk_status* st) {
  clear_status(st);
  if (n_failures) *n_failures = 0;
  if (int rc = gram_validate(m, len, dim, adaptive, order, tol, st)) return rc;
  if (nshards < 1 || shard >= nshards)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "gram_matrix: shard %zu out of range [0, %zu)", shard, nshards);
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  c.failures.clear();
  size_t t0 = 0, t1 = 0;
  sk_gram_shard_range(m, shard, nshards, &t0, &t1);
  for (size_t k = 0; k < m * m; ++k) {
    if (values) values[k] = std::numeric_limits<double>::quiet_NaN();
    if (orders) orders[k] = 0;
    if (pair_max) pair_max[k] = 0.0;
  }
  if (max_product) *max_product = 0.0;
  if (converged) *converged = 1;
  if (t1 == t0) return SK_OK;
  SK_CUDA(c.raw_x.ensure(m * len * dim * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_x.p, family, m * len * dim * sizeof(double)));
  GramCore g;
  const bool want_max = scan_products != 0;
  if (int rc = gram_core(c, c.raw_x.as<double>(), m, len, dim, adaptive, order, tol, flags, want_max,
                         pair_max != nullptr, t0, t1, g, st))
    return rc;
  double best = 0.0;
  for (size_t t = 0; t < g.pi.size(); ++t) {
    const size_t i = g.pi[t], j = g.pj[t];
    const double v = g.he[t] != ~0ull ? std::numeric_limits<double>::quiet_NaN() : g.hv[t];
    if (values) values[i * m + j] = values[j * m + i] = v;
    if (orders) orders[i * m + j] = orders[j * m + i] = g.ords[t];
    if (want_max) {
      double mr;
      std::memcpy(&mr, &g.hm[t], sizeof mr);
      if (pair_max) pair_max[i * m + j] = pair_max[j * m + i] = mr;
      if (best < mr) best = mr;
    }
    if (converged && !g.conv[t]) *converged = 0;
  }
  if (max_product) *max_product = best;
  if (n_failures) *n_failures = c.failures.size();
  return SK_OK;
}

int sk_gram_device(const double* d_family, size_t m, size_t len, size_t dim, int adaptive, int order, double tol,
                   uint32_t flags, int scan_products, size_t first, size_t last, double* d_matrix,
                   double* max_product, int* converged, size_t* n_failures, sk_status* st) {
  clear_status(st);
  if (n_failures) *n_failures = 0;
  if (max_product) *max_product = 0.0;
  if (converged) *converged = 1;
  if (int rc = gram_validate(m, len, dim, adaptive, order, tol, st)) return rc;
  if (first > last || last > m * (m + 1) / 2)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "gram_matrix: pair range [%zu, %zu) outside [0, %zu)", first,
                      last, m * (m + 1) / 2);
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Ctx& c = *cp;
  c.failures.clear();
  if (first == last) return SK_OK;
  GramCore g;
  const bool want_max = scan_products != 0;
  if (int rc = gram_core(c, d_family, m, len, dim, adaptive, order, tol, flags, want_max, false, first, last, g, st))
    return rc;
  // values (NaN for failed entries) into the mirrored matrix cells
  const size_t np = g.pi.size();
  SK_CUDA(c.gpairs.ensure(2 * np * sizeof(uint32_t)));
  SK_CUDA(cudaMemcpyAsync(c.gpairs.p, g.pi.data(), np * sizeof(uint32_t), cudaMemcpyHostToDevice, c.stream()));
  SK_CUDA(cudaMemcpyAsync(c.gpairs.as<uint32_t>() + np, g.pj.data(), np * sizeof(uint32_t), cudaMemcpyHostToDevice,
                          c.stream()));
  SK_CUDA(launch_scatter_gram(c.gpairs.as<uint32_t>(), c.gpairs.as<uint32_t>() + np, np, m, c.values.as<double>(),
                              c.err.as<unsigned long long>(), d_matrix, c.stream()));
  ++c.aux_launches;
  double best = 0.0;
  for (size_t t = 0; t < np; ++t) {
    if (want_max) {
      double mr;
      std::memcpy(&mr, &g.hm[t], sizeof mr);
      if (best < mr) best = mr;
    }
    if (converged && !g.conv[t]) *converged = 0;
  }
  if (max_product) *max_product = best;
  if (n_failures) *n_failures = c.failures.size();
  SK_CUDA(cudaStreamSynchronize(c.stream()));  // g's host arrays back the pair-list upload
  return SK_OK;
}

size_t sk_gram_failures(sk_gram_failure* out, size_t cap) {
  sk_status st;
  Ctx* c = nullptr;
  if (get_ctx(&c, &st)) return 0;
  const size_t n = std::min(cap, c->failures.size());
  if (out) std::copy(c->failures.begin(), c->failures.begin() + n, out);
  return n;
}

// ------------------------------------------------------ multi-GPU strips
static int np_of(int order) { return col_stride(order <= kMaxRegOrder ? order : 0); }

int sk_strip_bands(size_t ly, int order, size_t* bands) {
  if (ly < 2 || order < 1 || order > kMaxOrder) return SK_INVALID_ARGUMENT;
  const size_t band_rows = 32 * static_cast<size_t>(rows_per_lane(order <= kMaxRegOrder ? order : 0));
  *bands = (ly - 1 + band_rows - 1) / band_rows;
  return SK_OK;
}

int sk_exchange_alloc(size_t lx, int order, size_t rounds, void** abuf, void** prog, sk_status* st) {
  clear_status(st);
  if (lx < 2 || order < 1 || order > kMaxOrder || rounds < 1)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "exchange: bad length/order/rounds");
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  const size_t bytes = rounds * (lx - 1) * np_of(order) * sizeof(double);
  SK_CUDA(cudaMalloc(abuf, bytes));
  SK_CUDA(cudaMalloc(prog, rounds * kXProg * sizeof(unsigned long long)));
  // zeroed on the context's (non-blocking) stream and waited for: a legacy-
  // stream memset would not be ordered against the sweeps
  SK_CUDA(cudaMemsetAsync(*prog, 0, rounds * kXProg * sizeof(unsigned long long), cp->stream()));
  SK_CUDA(cudaStreamSynchronize(cp->stream()));
  return SK_OK;
}

int sk_exchange_reset(void* prog, size_t rounds, sk_status* st) {
  clear_status(st);
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  SK_CUDA(cudaMemsetAsync(prog, 0, rounds * kXProg * sizeof(unsigned long long), cp->stream()));
  SK_CUDA(cudaStreamSynchronize(cp->stream()));
  return SK_OK;
}

int sk_exchange_free(void* abuf, void* prog) {
  if (abuf) cudaFree(abuf);
  if (prog) cudaFree(prog);
  return SK_OK;
}

int sk_ipc_handle(void* dptr, void* handle64, sk_status* st) {
  clear_status(st);
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  cudaIpcMemHandle_t h;
  SK_CUDA(cudaIpcGetMemHandle(&h, dptr));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle64, &h, sizeof h);
  return SK_OK;
}

int sk_ipc_open(const void* handle64, void** dptr, sk_status* st) {
  clear_status(st);
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  SK_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

int sk_ipc_close(void* dptr) {
  cudaIpcCloseMemHandle(dptr);
  return SK_OK;
}

// In-process alternative to IPC: let the calling thread's device read and
// write `peer`'s memory directly (one process driving several GPUs).
int sk_enable_peer_access(int peer, sk_status* st) {
  clear_status(st);
  Ctx* c = nullptr;
  if (int rc = get_ctx(&c, st)) return rc;
  if (peer == c->device) return SK_OK;
  int can = 0;
  SK_CUDA(cudaDeviceCanAccessPeer(&can, c->device, peer));
  if (!can)
    return set_status(st, SK_CUDA_ERROR, 0, 0, "GPU %d cannot access GPU %d's memory (no peer path)", c->device, peer);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SK_OK;
  }
  SK_CUDA(e);
  return SK_OK;
}

int sk_strip_plan(size_t ly, int order, size_t gpus, size_t rank, size_t block, size_t* owned_bands,
                  size_t* rounds, size_t* in_rounds) {
  size_t bands = 0;
  if (gpus < 1 || rank >= gpus || block < 1 || sk_strip_bands(ly, order, &bands) != SK_OK) return SK_INVALID_ARGUMENT;
  const StripPlan pl = strip_plan(bands, gpus, rank, block);
  if (owned_bands) *owned_bands = pl.owned_bands;
  if (rounds) *rounds = pl.rounds;
  if (in_rounds) *in_rounds = pl.in_rounds;
  return SK_OK;
}

// Shared by sk_propagate_strip (one GPU of a multi-GPU pipeline) and
// sk_propagate_split (every GPU of the pipeline emulated in ONE launch on one
// GPU: gpus = 1, every block boundary still routed through an exchange area).
static int strip_launch(Ctx& c, const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order,
                        uint32_t flags, const Strip& s, double* value, double* diag, sk_status* st) {
  const size_t ld = inc_ld(dim);
  SK_CUDA(c.raw_x.ensure(lx * dim * sizeof(double)));
  SK_CUDA(c.raw_y.ensure(ly * dim * sizeof(double)));
  SK_CUDA(c.xinc.ensure(lx * ld * sizeof(double)));
  SK_CUDA(c.yinc.ensure(ly * ld * sizeof(double)));
  SK_CUDA(c.values.ensure(sizeof(double)));
  SK_CUDA(h2d(c, c.raw_x.p, x, lx * dim * sizeof(double)));
  SK_CUDA(h2d(c, c.raw_y.p, y, ly * dim * sizeof(double)));
  SK_CUDA(launch_increments(c.raw_x.as<double>(), 1, lx, dim, ld, c.xinc.as<double>(), c.stream()));
  SK_CUDA(launch_increments(c.raw_y.as<double>(), 1, ly, dim, ld, c.yinc.as<double>(), c.stream()));
  c.aux_launches += 2;
  SK_CUDA(c.err.ensure(sizeof(unsigned long long)));
  SK_CUDA(cudaMemsetAsync(c.err.p, 0xff, sizeof(unsigned long long), c.stream()));
  SK_CUDA(cudaMemsetAsync(c.values.p, 0xff, sizeof(double), c.stream()));
  const size_t nd = std::min(lx, ly) - 1;
  double* d_diag = nullptr;
  if (diag) {
    SK_CUDA(c.diag.ensure(nd * sizeof(double)));
    d_diag = c.diag.as<double>();
    SK_CUDA(cudaMemsetAsync(d_diag, 0xff, nd * sizeof(double), c.stream()));
  }
  PairSet ps{c.xinc.as<double>(), c.yinc.as<double>(), lx * ld, ly * ld, static_cast<int>(ly - 1),
             static_cast<int>(lx - 1), static_cast<int>(dim), static_cast<int>(ld)};
  Outputs o{c.values.as<double>(), c.err.as<unsigned long long>(), nullptr, nullptr, d_diag, lx * ly, nd};
  std::vector<uint32_t> zero(1, 0);
  if (int rc = run_sweeps(c, ps, zero, zero, zero, order, flags | kFlagAllTotals, o, st, s)) return rc;
  unsigned long long key = ~0ull;
  SK_CUDA(cudaMemcpyAsync(&key, c.err.p, sizeof key, cudaMemcpyDeviceToHost, c.stream()));
  double v = std::numeric_limits<double>::quiet_NaN();
  SK_CUDA(cudaMemcpyAsync(&v, c.values.p, sizeof v, cudaMemcpyDeviceToHost, c.stream()));
  if (diag) SK_CUDA(cudaMemcpyAsync(diag, d_diag, nd * sizeof(double), cudaMemcpyDeviceToHost, c.stream()));
  SK_CUDA(cudaStreamSynchronize(c.stream()));
  if (key != ~0ull)
    return decode_err(key, st, device_delta(c, c.xinc.as<double>(), c.yinc.as<double>(), ld, dim, key));
  if (value) *value = v;
  return SK_OK;
}

// One GPU's share of a long pair over `gpus` GPUs (block-cyclic: blocks of
// `block` bands, GPU `rank` sweeps blocks rank, rank + gpus, ...).  in_abuf /
// in_prog: this GPU's exchange area (sk_exchange_alloc with in_rounds of
// sk_strip_plan), written by GPU rank - 1 (mod gpus); out_abuf / out_prog:
// GPU rank + 1's area (peer pointers, sk_ipc_open or peer access).  All GPUs
// of a pair run concurrently.  *value is written by the GPU that owns the last
// band; diag (optional, min(lx,ly)-1 entries) receives this GPU's knots.
int sk_propagate_strip(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order, uint32_t flags,
                       size_t gpus, size_t rank, size_t block, const void* in_abuf, const void* in_prog,
                       void* out_abuf, void* out_prog, double* value, double* diag, sk_status* st) {
  clear_status(st);
  size_t bands = 0;
  if (dim < 1 || sk_strip_bands(ly, order, &bands) != SK_OK || lx < 2)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate_strip: bad arguments");
  if (gpus < 1 || rank >= gpus || block < 1)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate_strip: rank %zu of %zu GPUs, block %zu", rank, gpus,
                      block);
  const size_t nblocks = (bands + block - 1) / block;
  const StripPlan pl = strip_plan(bands, gpus, rank, block);
  // blocks other than the last hand up; whether this GPU sends / receives
  bool sends = false;
  for (size_t k = rank; k + 1 < nblocks; k += gpus) sends = true;
  if ((pl.in_rounds > 0) != (in_abuf != nullptr && in_prog != nullptr) ||
      (sends && gpus > 1) != (out_abuf != nullptr && out_prog != nullptr))
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate_strip: exchange buffers do not match the plan");
  Ctx* cp = nullptr;
  if (int rc = get_ctx(&cp, st)) return rc;
  Strip s;
  s.gpus = static_cast<int>(gpus);
  s.rank = static_cast<int>(rank);
  s.block = static_cast<int>(block);
  s.exch = gpus > 1;
  s.xin_abuf = static_cast<const double*>(in_abuf);
  s.xin_prog = static_cast<const unsigned long long*>(in_prog);
  s.xout_abuf = static_cast<double*>(out_abuf);
  s.xout_prog = static_cast<unsigned long long*>(out_prog);
  double v = std::numeric_limits<double>::quiet_NaN();
  if (int rc = strip_launch(*cp, x, lx, y, ly, dim, order, flags, s, &v, diag, st)) return rc;
  if ((nblocks - 1) % gpus == rank && value) *value = v;
  return SK_OK;
}

// One-GPU emulation of the strip pipeline: ONE launch sweeps every band of
// all `gpus` virtual GPUs (global band order), with the block-cyclic layout's
// column buffers and exchange areas per virtual GPU and every block boundary
// handed over through an exchange area with system-scope release/acquire,
// exactly as between GPUs.  Used to test the multi-GPU path on one GPU
// (strips on one GPU may not run as separate launches that wait on each other).
int sk_propagate_split(const double* x, size_t lx, const double* y, size_t ly, size_t dim, int order, uint32_t flags,
                       size_t gpus, size_t block, double* value, sk_status* st) {
  clear_status(st);
  size_t bands = 0;
  if (dim < 1 || sk_strip_bands(ly, order, &bands) != SK_OK || lx < 2 || block < 1 || block >= bands || gpus < 1)
    return set_status(st, SK_INVALID_ARGUMENT, 0, 0, "propagate_split: block outside [1, bands) or no GPUs");
  const size_t nblocks = (bands + block - 1) / block;
  const size_t xrounds = (nblocks + gpus - 1) / gpus;
  void *xa = nullptr, *xp = nullptr;
  if (int rc = sk_exchange_alloc(lx, order, gpus * xrounds, &xa, &xp, st)) return rc;
  Ctx* cp = nullptr;
  int rc = get_ctx(&cp, st);
  if (rc == SK_OK) {
    Strip s;
    s.gpus = static_cast<int>(gpus);
    s.rank = 0;
    s.block = static_cast<int>(block);
    s.exch = true;
    s.emul = true;
    s.xin_abuf = static_cast<const double*>(xa);
    s.xout_abuf = static_cast<double*>(xa);
    s.xin_prog = static_cast<const unsigned long long*>(xp);
    s.xout_prog = static_cast<unsigned long long*>(xp);
    rc = strip_launch(*cp, x, lx, y, ly, dim, order, flags, s, value, nullptr, st);
  }
  sk_exchange_free(xa, xp);
  return rc;
}

int sk_all_finite(const double* v, size_t n) {
  // exponent all ones <=> inf or NaN; OR-reduce per chunk (vectorises)
  constexpr uint64_t kExp = 0x7ff0000000000000ull;
  auto scan = [v](size_t b, size_t e) {
    uint64_t bad = 0;
    for (size_t k = b; k < e; ++k) {
      uint64_t u;
      std::memcpy(&u, v + k, sizeof u);
      bad |= static_cast<uint64_t>((u & kExp) == kExp);
    }
    return bad == 0;
  };
  constexpr size_t kPerThread = size_t{1} << 20;
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>({hw, 16, (n + kPerThread - 1) / kPerThread});
  if (nt <= 1) return scan(0, n) ? 1 : 0;
  std::vector<char> ok(nt, 1);
  std::vector<std::thread> pool;
  const size_t chunk = (n + nt - 1) / nt;
  for (size_t t = 1; t < nt; ++t)
    pool.emplace_back([&, t] { ok[t] = scan(std::min(n, t * chunk), std::min(n, (t + 1) * chunk)); });
  ok[0] = scan(0, std::min(n, chunk));
  for (auto& th : pool) th.join();
  return std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; }) ? 1 : 0;
}

int sk_gram_shard_range(size_t m, size_t shard, size_t nshards, size_t* first, size_t* last) {
  if (nshards < 1 || shard >= nshards) return SK_INVALID_ARGUMENT;
  const size_t total = m * (m + 1) / 2;
  *first = total * shard / nshards;
  *last = total * (shard + 1) / nshards;
  return SK_OK;
}

int sk_stats_enable(int enable) {
  sk_status st;
  Ctx* c = nullptr;
  if (get_ctx(&c, &st)) return st.code;
  c->stats_on = enable != 0;
  return SK_OK;
}

int sk_stats_reset(void) {
  sk_status st;
  Ctx* c = nullptr;
  if (get_ctx(&c, &st)) return st.code;
  cudaStreamSynchronize(c->stream());
  for (auto& r : c->stats) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  c->stats.clear();
  c->sweep_launches = c->aux_launches = c->literal_rechecks = 0;
  c->done_ms = c->done_tiles = c->done_flops = 0.0;
  return SK_OK;
}

int sk_stats_get(sk_stats* out) {
  sk_status st;
  Ctx* c = nullptr;
  if (get_ctx(&c, &st)) return st.code;
  for (auto& r : c->stats) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->done_ms += ms;
    c->done_tiles += r.tiles;
    c->done_flops += r.flops;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  c->stats.clear();
  out->sweep_launches = c->sweep_launches;
  out->aux_launches = c->aux_launches;
  out->sweep_ms = c->done_ms;
  out->tiles = c->done_tiles;
  out->tile_flops = c->done_flops;
  out->literal_rechecks = c->literal_rechecks;
  return SK_OK;
}

int sk_release(void) {
  if (t_ctx) {
    cudaStreamSynchronize(t_ctx->stream());
    t_ctx.reset();
  }
  return SK_OK;
}

}  // extern "C"
