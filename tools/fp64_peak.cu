// FP64 peak microbenchmark (measurement tooling, not product code).
// (1) DFMA throughput: independent FMA chains, 148 x k CTAs; (2) the P2P exponential core
// (sincos of a double) for reference.  Prints TFLOP/s (2 flops per DFMA) and clocks used.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int occ : {4, 8}) {
    int blocks = sms * occ;
    dfma_loop<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 16 * 8;
    printf("{\"test\": \"dfma\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965\": %.2f}\n",
           occ, ms, 2 * fmas / (ms * 1e-3) / 1e12, fmas / (ms * 1e-3) / (sms * 1.965e9));
  }
  return 0;
}
