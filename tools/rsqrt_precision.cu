// Max relative error of rsqrt.approx.ftz.f64 (MUFU.RSQ64H seed) over a log-uniform sample of
// r2 in [1e-6, 1e12], and of one quadratic / cubic Newton step (decides the P2P rsqrt recipe).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(double *err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = -6.0 + 18.0 * (double)i / (double)n;
  double r2 = pow(10.0, t);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  double ex = 1.0 / sqrt(r2);
  double e = fma(-r2, y * y, 1.0);
  double yq = fma(y * e, 0.5, y);
  double yc = fma(y * e, fma(e, 0.375, 0.5), y);
  err[3 * i] = fabs(y / ex - 1.0);
  err[3 * i + 1] = fabs(yq / ex - 1.0);
  err[3 * i + 2] = fabs(yc / ex - 1.0);
}
int main() {
  const int n = 1 << 22;
  double *d, *h = new double[3 * n];
  cudaMalloc(&d, 3 * n * sizeof(double));
  k<<<(n + 255) / 256, 256>>>(d, n);
  cudaMemcpy(h, d, 3 * n * sizeof(double), cudaMemcpyDeviceToHost);
  double m[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) m[j] = fmax(m[j], h[3 * i + j]);
  printf("rsqrt.approx.f64 max rel err %.3e (2^%.1f); quadratic Newton %.3e; cubic Newton %.3e\n", m[0],
         log2(m[0]), m[1], m[2]);
  return 0;
}
