// One translation unit per truncation order: compiled once per SK_N value
// (Makefile) so the 17 x 5 x 2 sweep instantiations build in parallel.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sk_sweep.cuh"

#ifndef SK_N
#error "SK_N must be defined"
#endif

namespace skb {

template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
static size_t smem_bytes() {
  return static_cast<size_t>(sweep_smem_doubles(N, DP, LIT)) * sizeof(double);
}

template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
static cudaError_t prepare() {
  // function attributes are per device: set them once per device
  static std::atomic<unsigned long long> done_mask{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const size_t smem = smem_bytes<N, DP, EXACT, EXTRAS, LIT>();
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(sweep_kernel<N, DP, EXACT, EXTRAS, LIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  // the whole unified L1/shared array as shared memory: residency is set by
  // registers and the per-warp stage, never by a smaller default carveout
  // (the sweep reads global memory only through L2-bypassing cp.async)
  e = cudaFuncSetAttribute(sweep_kernel<N, DP, EXACT, EXTRAS, LIT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
static cudaError_t launch_one(int grid, cudaStream_t stream, const SweepParams& P) {
  cudaError_t e = prepare<N, DP, EXACT, EXTRAS, LIT>();
  if (e != cudaSuccess) return e;
#ifdef SK_PROFILE_WAITS
  {
    static const unsigned zero = 0;
    cudaMemcpyToSymbolAsync(g_tidx, &zero, sizeof zero, 0, cudaMemcpyHostToDevice, stream);
    void* tp = nullptr;
    cudaGetSymbolAddress(&tp, g_utrace);
    cudaMemsetAsync(tp, 0, kTraceUnits * 4 * sizeof(unsigned long long), stream);
  }
#endif
  // compact table-mode layout (slot_stride): sweep warps only, the slots
  // packed, and at least kTableCtaSmem requested so that two sweep CTAs never
  // share an SM (one latency-bound sweep warp per sub-partition) while two
  // GEMM CTAs still fit beside one
  int threads = sweep_warps(N, DP) * 32;
  size_t smem = smem_bytes<N, DP, EXACT, EXTRAS, LIT>();
  if (DP == 0 && P.slot_stride > 0) {
    threads = rho_bands(N) * 32;
    smem = std::max(static_cast<size_t>(rho_bands(N)) * P.slot_stride * sizeof(double), kTableCtaSmem);
  }
  sweep_kernel<N, DP, EXACT, EXTRAS, LIT><<<grid, threads, smem, stream>>>(P);
#ifdef SK_PROFILE_WAITS
  if (const char* path = std::getenv("SK_UTRACE")) {
    static std::vector<unsigned long long> h(kTraceUnits * 4);
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h.data(), g_utrace, h.size() * sizeof(unsigned long long));
    if (FILE* f = std::fopen(path, "wb")) {
      std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      std::fclose(f);
    }
  }
#endif
  return cudaGetLastError();
}

template <int N, int DP, bool EXACT, bool EXTRAS, bool LIT = false>
static cudaError_t occupancy_one(int* blocks_per_sm) {
  cudaError_t e = prepare<N, DP, EXACT, EXTRAS, LIT>();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sweep_kernel<N, DP, EXACT, EXTRAS, LIT>,
                                                       sweep_warps(N, DP) * 32, smem_bytes<N, DP, EXACT, EXTRAS, LIT>());
}

#define SK_CAT2(a, b) a##b
#define SK_CAT(a, b) SK_CAT2(a, b)

// Variants: N > 0 -> (exact, extras) in {(0,0), (1,0), (0,1)}; (1,1) maps to
// (1,0) + ... never requested (grids never ask for max|rho|).  N = 0 (literal
// kernel) always runs the fully general <true, true> variant.
#if SK_N > 0
#define SK_VAR(FN, DPV, ...)                                                      \
  (extras ? FN<SK_N, DPV, false, true>(__VA_ARGS__)                               \
          : (exact ? FN<SK_N, DPV, true, false>(__VA_ARGS__) : FN<SK_N, DPV, false, false>(__VA_ARGS__)))
#else
#define SK_VAR(FN, DPV, ...) FN<SK_N, DPV, true, true>(__VA_ARGS__)
#endif

#define SK_DP_SWITCH(FN, ...)                    \
  switch (dp) {                                  \
    case 0: return SK_VAR(FN, 0, __VA_ARGS__);   \
    case 2: return SK_VAR(FN, 2, __VA_ARGS__);   \
    case 4: return SK_VAR(FN, 4, __VA_ARGS__);   \
    case 8: return SK_VAR(FN, 8, __VA_ARGS__);   \
    case 16: return SK_VAR(FN, 16, __VA_ARGS__); \
    default: return cudaErrorInvalidValue;       \
  }

// Literal arithmetic at this compile-time order (strict-corner re-sweeps of
// register-kernel pairs): instantiated for the order every Brownian config
// runs at (N = 8); other orders re-sweep with the runtime-order kernel N = 0.
#if SK_N == 8
#define SK_LIT_SWITCH(FN, ...)                                           \
  switch (dp) {                                                          \
    case 0: return FN<SK_N, 0, true, true, true>(__VA_ARGS__);           \
    case 2: return FN<SK_N, 2, true, true, true>(__VA_ARGS__);           \
    case 4: return FN<SK_N, 4, true, true, true>(__VA_ARGS__);           \
    case 8: return FN<SK_N, 8, true, true, true>(__VA_ARGS__);           \
    case 16: return FN<SK_N, 16, true, true, true>(__VA_ARGS__);         \
    default: return cudaErrorInvalidValue;                               \
  }
#else
#define SK_LIT_SWITCH(FN, ...) return cudaErrorInvalidValue;
#endif

cudaError_t SK_CAT(sweep_launch_n, SK_N)(int dp, bool exact, bool extras, bool literal, int grid, cudaStream_t stream,
                                         const SweepParams& P) {
  if (literal) SK_LIT_SWITCH(launch_one, grid, stream, P)
  SK_DP_SWITCH(launch_one, grid, stream, P)
}

cudaError_t SK_CAT(sweep_occupancy_n, SK_N)(int dp, bool exact, bool extras, bool literal, int* blocks_per_sm) {
  if (literal) SK_LIT_SWITCH(occupancy_one, blocks_per_sm)
  SK_DP_SWITCH(occupancy_one, blocks_per_sm)
}

}  // namespace skb
