// Dispatch from a runtime order to the per-order sweep instantiations
// (sk_sweep_inst.cu compiled once per SK_N; weak so that experimental builds
// with a subset of orders still link).
#include <cuda_runtime.h>

#include "sk_internal.h"
#include "sk_sweep.cuh"

namespace skb {

#define SK_DECL(n)                                                                                          \
  __attribute__((weak)) cudaError_t sweep_launch_n##n(int dp, bool exact, bool extras, bool literal, int grid, \
                                                      cudaStream_t stream, const SweepParams& P);           \
  __attribute__((weak)) cudaError_t sweep_occupancy_n##n(int dp, bool exact, bool extras, bool literal,      \
                                                         int* blocks_per_sm);
SK_DECL(0) SK_DECL(1) SK_DECL(2) SK_DECL(3) SK_DECL(4) SK_DECL(5) SK_DECL(6) SK_DECL(7) SK_DECL(8)
SK_DECL(9) SK_DECL(10) SK_DECL(11) SK_DECL(12) SK_DECL(13) SK_DECL(14) SK_DECL(15) SK_DECL(16)
#undef SK_DECL

#define SK_CASE(n, fn, ...) \
  case n: return fn##n ? fn##n(__VA_ARGS__) : cudaErrorInvalidValue;
#define SK_ALL(fn, ...)                                                                                     \
  SK_CASE(0, fn, __VA_ARGS__) SK_CASE(1, fn, __VA_ARGS__) SK_CASE(2, fn, __VA_ARGS__)                      \
  SK_CASE(3, fn, __VA_ARGS__) SK_CASE(4, fn, __VA_ARGS__) SK_CASE(5, fn, __VA_ARGS__)                      \
  SK_CASE(6, fn, __VA_ARGS__) SK_CASE(7, fn, __VA_ARGS__) SK_CASE(8, fn, __VA_ARGS__)                      \
  SK_CASE(9, fn, __VA_ARGS__) SK_CASE(10, fn, __VA_ARGS__) SK_CASE(11, fn, __VA_ARGS__)                    \
  SK_CASE(12, fn, __VA_ARGS__) SK_CASE(13, fn, __VA_ARGS__) SK_CASE(14, fn, __VA_ARGS__)                   \
  SK_CASE(15, fn, __VA_ARGS__) SK_CASE(16, fn, __VA_ARGS__)

cudaError_t sweep_launch(int n_template, int dp, bool exact, bool extras, bool literal, int grid, cudaStream_t stream,
                         const SweepParams& P) {
  switch (n_template) {
    SK_ALL(sweep_launch_n, dp, exact, extras, literal, grid, stream, P)
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t sweep_occupancy(int n_template, int dp, bool exact, bool extras, bool literal, int* blocks_per_sm) {
  switch (n_template) {
    SK_ALL(sweep_occupancy_n, dp, exact, extras, literal, blocks_per_sm)
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace skb
