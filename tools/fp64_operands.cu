// FP64 pipe throughput vs the number of distinct register operands per instruction
// (measurement tooling, not product code).  Each test runs 8 independent chains per thread,
// 16 x 8 instructions per loop trip, 12 warps / SM (the P2P kernel's occupancy) and reports
// FP64 instructions per clock per SM at the given SM clock (argv[1], MHz).
//   fma3   x_i = fma(a_j, b_k, x_i)      three distinct registers
//   fma3r  x_i = fma(A, b_i, x_i)        A shared by consecutive instructions (operand reuse)
//   fma2c  x_i = fma(x_i, b_i, C)        two registers + a constant-bank operand
//   fma2i  x_i = fma(x_i, b_i, 1.0)      two registers + an immediate
//   fma1   x_i = fma(x_i, A, C)          one register (+ reuse/constant)
//   dadd   x_i = x_i + b_i               two registers
//   dmul   x_i = x_i * b_i               two registers
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int T>
__global__ void loop(double *out, int iters, const double *in, double C) {
  double a[8], b[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[i] + threadIdx.x, b[i] = in[8 + i] - threadIdx.x, x[i] = in[16 + i];
  const double A = a[0] * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (T == 0) x[i] = fma(a[(i + u) & 7], b[(i + 3 * u) & 7], x[i]);
        if (T == 1) x[i] = fma(A, b[(i + u) & 7], x[i]);
        if (T == 2) x[i] = fma(x[i], b[(i + u) & 7], C);
        if (T == 3) x[i] = fma(x[i], b[(i + u) & 7], 1.0);
        if (T == 4) x[i] = fma(x[i], A, C);
        if (T == 5) x[i] = x[i] + b[(i + u) & 7];
        if (T == 6) x[i] = x[i] * b[(i + u) & 7];
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <int T>
static void run(const char *name, double *o, const double *in, int sms, double mhz) {
  const int blocks = sms * 3, threads = 128, iters = 20000;
  loop<T><<<blocks, threads>>>(o, 100, in, 0.9999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    loop<T><<<blocks, threads>>>(o, iters, in, 0.9999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double f = (double)blocks * threads * iters * 16 * 8;
  printf("{\"test\": \"%s\", \"ms\": %.3f, \"fp64_inst_per_clk_sm\": %.2f}\n", name, best, f / (best * 1e-3) / (sms * mhz * 1e6));
}

int main(int argc, char **argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *in, *o;
  cudaMalloc(&in, 24 * 8), cudaMalloc(&o, 8);
  double hi[24];
  for (int i = 0; i < 24; ++i) hi[i] = 0.999 + 1e-4 * i;
  cudaMemcpy(in, hi, sizeof(hi), cudaMemcpyHostToDevice);
  run<0>("fma3", o, in, sms, mhz);
  run<1>("fma3r", o, in, sms, mhz);
  run<2>("fma2c", o, in, sms, mhz);
  run<3>("fma2i", o, in, sms, mhz);
  run<4>("fma1", o, in, sms, mhz);
  run<5>("dadd", o, in, sms, mhz);
  run<6>("dmul", o, in, sms, mhz);
  return 0;
}
