// DFMA issue rate vs operand sourcing on B200: how many distinct 64-bit
// register operands a DFMA can read per issue (register-file bank limits),
// and whether constant-bank operands relieve it.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double c_k[16] = {1.0000001, 0.9999999, 1.0000002, 0.9999998, 1.0000003, 0.9999997, 1.0000004, 0.9999996,
                               1.0000005, 0.9999995, 1.0000006, 0.9999994, 1.0000007, 0.9999993, 1.0000008, 0.9999992};

// 8 chains, each DFMA reads acc[c], x[c], y[c]: three distinct register pairs
__global__ void distinct3(double* out, int iters) {
  double acc[8], x[8], y[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = threadIdx.x + c;
    x[c] = 1.0 + 1e-9 * c + threadIdx.x * 1e-13;
    y[c] = 1e-12 * (c + 1) + threadIdx.x * 1e-15;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], x[c], y[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], y[c], acc[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + x[c];
  if (s == 1.2345) out[0] = s;
}

// acc[c] = fma(acc[c], c_k[c], y[c]): one operand from the constant bank
__global__ void const_operand(double* out, int iters) {
  double acc[8], y[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = threadIdx.x + c;
    y[c] = 1e-12 * (c + 1) + threadIdx.x * 1e-15;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], c_k[c], y[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = fma(y[c], c_k[c + 8], acc[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + y[c];
  if (s == 1.2345) out[0] = s;
}

// acc[c] = fma(x[c], p, acc[c]) with one shared operand p (reuse)
__global__ void shared_operand(double* out, int iters, double p) {
  double acc[8], x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = threadIdx.x + c;
    x[c] = 1.0 + 1e-9 * c;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(x[c], p, acc[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(acc[c], p, x[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + x[c];
  if (s == 1.2345) out[0] = s;
}

// 3 distinct vector registers, with the multiplier a per-lane value (like a
// constant hoisted into a vector register)
__global__ void reg_const(double* out, int iters) {
  double acc[8], y[8], k[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = threadIdx.x + c;
    y[c] = 1e-12 * (c + 1) + threadIdx.x * 1e-15;
    k[c] = 1.0 + 1e-9 * c + threadIdx.x * 1e-13;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], k[c], y[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) y[c] = fma(y[c], k[7 - c], acc[c]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + y[c];
  if (s == 1.2345) out[0] = s;
}

// conv pattern: acc[c] = fma(x[c], pv, acc[c]) with pv a per-lane register
// shared by 8 consecutive DFMAs (operand reuse cache), 3 register operands
__global__ void shared_reg(double* out, int iters) {
  double acc[8], x[8];
  double pv = 1.0 + threadIdx.x * 1e-13, pw = 1.0 - threadIdx.x * 1e-13;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = threadIdx.x + c;
    x[c] = 1.0 + 1e-9 * c;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(x[c], pv, acc[c]);
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(acc[c], pw, x[c]);
    const double t = pv;
    pv = pw;
    pw = t;
  }
  double s = pv + pw;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c] + x[c];
  if (s == 1.2345) out[0] = s;
}

template <class F>
void run(const char* name, F launch, double flops_per_launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("%-16s %.2f TFLOP/s\n", name, flops_per_launch / ms / 1e9);
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, tpb = 256, blocks = sms * 8;
  const double fl = 2.0 * 16 * iters * (double)blocks * tpb;
  run("distinct3", [&] { distinct3<<<blocks, tpb>>>(out, iters); }, fl);
  run("reg_const", [&] { reg_const<<<blocks, tpb>>>(out, iters); }, fl);
  run("const_operand", [&] { const_operand<<<blocks, tpb>>>(out, iters); }, fl);
  run("shared_reg", [&] { shared_reg<<<blocks, tpb>>>(out, iters); }, fl);
  run("shared_operand", [&] { shared_operand<<<blocks, tpb>>>(out, iters, 1.0000001); }, fl);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
