// P2P inner-loop ablation microbenchmark (measurement tooling, not product code).
// Re-states the symmetric P2P kernel body (kernels_points.cu p2p_sym_kernel, PT targets per
// thread, 128 threads, e^{ix} table in shared memory, systolic column shuffles) on synthetic
// items and removes one ingredient at a time, to find what holds the FP64 pipe below its
// DFMA-only rate:
//   V_NOTAB   table entry from integer moves of k (no LDS, no bank conflicts)
//   V_NOMUFU  rsqrt seed from integer ops (no XU instruction)
//   V_NOSHFL  column accumulators not passed between lanes (no SHFL)
// plus a DFMA chain test with three distinct register operands per DFMA.
// Output: one JSON line per variant, pair evaluations / s and FP64 lane-ops / clk / SM
// (33 FP64 instructions per evaluation as compiled; clock from nvidia-smi supplied on argv).
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

constexpr int TAB = 2048;
constexpr int TPB = 128;
constexpr double kMagic = 6755399441055744.0;
constexpr double kH = 6.283185307179586476925286766559 / TAB;
constexpr double kS1 = kH, kS3 = -kH * kH * kH / 6.0;
constexpr double kC2 = -kH * kH / 2.0, kC4 = kH * kH * kH * kH / 24.0;

enum { V_NOTAB = 1, V_NOMUFU = 2, V_NOSHFL = 4, V_TWOACC = 8, V_MACORD = 16 };

template <int V>
__device__ __forceinline__ double rsq(double r2) {
  double y;
  if (V & V_NOMUFU) {
    y = __hiloint2double(0x5FE6EB50 - (__double2hiint(r2) >> 1), 0);
  } else {
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  }
  const double e = fma(-r2, y * y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}

template <int V>
__device__ __forceinline__ double2 green(double tx, double ty, double tz, double xs, double ys, double zs,
                                         const double2 *tab) {
  const double dx = tx - xs, dy = ty - ys, dz = tz - zs;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ri = rsq<V>(r2);
  const double t = fma(r2, ri, kMagic);
  const int k = __double2loint(t);
  const double r = fma(r2, ri, -(t - kMagic));
  const double rr = r * r;
  const double s = r * fma(rr, kS3, kS1);
  const double c = fma(rr, fma(rr, kC4, kC2), 1.0);
  double2 e;
  if (V & V_NOTAB) e = make_double2(__hiloint2double(0x3FE00000, k), __hiloint2double(0x3FD00000, k));
  else e = tab[k & (TAB - 1)];
  const double2 g = make_double2(fma(e.x, c, -e.y * s), fma(e.x, s, e.y * c));
  return make_double2(g.x * ri, g.y * ri);
}

template <int V, int PT, int MINB, int UNR = 2>
__global__ void __launch_bounds__(TPB, MINB) sym_kernel(const double *ux, const double *uy, const double *uz,
                                                        const double2 *q, int nt, int ns, double2 *out) {
  __shared__ double2 tab[TAB];
  __shared__ double sx[TPB], sy[TPB], sz[TPB];
  __shared__ double2 sq[TPB];
  __shared__ double2 col[TPB / 32][TPB];
  for (int t = threadIdx.x; t < TAB; t += TPB) {
    double s, c;
    sincospi((double)t / (TAB / 2), &s, &c);
    tab[t] = make_double2(c, s);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * nt;           // targets of this item
  const int64_t s0 = (int64_t)blockIdx.x * ns + 7777;    // sources of this item (another range)
  double tx[PT], ty[PT], tz[PT], ar[PT], ai[PT];
  double2 tq[PT];
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int64_t i = t0 + threadIdx.x + p * TPB;
    tx[p] = ux[i], ty[p] = uy[i], tz[p] = uz[i];
    tq[p] = q[i];
    ar[p] = ai[p] = 0.0;
  }
  double2 csum = make_double2(0.0, 0.0);
  for (int c0 = 0; c0 < ns; c0 += TPB) {
    __syncthreads();
    sx[threadIdx.x] = ux[s0 + c0 + threadIdx.x];
    sy[threadIdx.x] = uy[s0 + c0 + threadIdx.x];
    sz[threadIdx.x] = uz[s0 + c0 + threadIdx.x];
    sq[threadIdx.x] = q[s0 + c0 + threadIdx.x];
    __syncthreads();
    for (int blk = 0; blk < TPB / 32; ++blk) {
      const int base = blk << 5;
      double cr = 0.0, ci = 0.0, cr2 = 0.0, ci2 = 0.0;
#pragma unroll UNR
      for (int u = 0; u < 32; ++u) {
        const int s = base + ((lane + u) & 31);
        const double xs = sx[s], ys = sy[s], zs = sz[s];
        const double2 qs = sq[s];
        if (V & V_MACORD) {
          double2 g[PT];
#pragma unroll
          for (int p = 0; p < PT; ++p) g[p] = green<V>(tx[p], ty[p], tz[p], xs, ys, zs, tab);
#pragma unroll
          for (int p = 0; p < PT; ++p) ar[p] = fma(qs.x, g[p].x, ar[p]);
#pragma unroll
          for (int p = 0; p < PT; ++p) ai[p] = fma(qs.y, g[p].x, ai[p]);
#pragma unroll
          for (int p = 0; p < PT; ++p) ai[p] = fma(qs.x, g[p].y, ai[p]);
#pragma unroll
          for (int p = 0; p < PT; ++p) ar[p] = fma(-qs.y, g[p].y, ar[p]);
#pragma unroll
          for (int p = 0; p < PT; ++p) {
            cr = fma(g[p].x, tq[p].x, cr);
            ci = fma(g[p].x, tq[p].y, ci);
            ci = fma(g[p].y, tq[p].x, ci);
            cr = fma(-g[p].y, tq[p].y, cr);
          }
        } else
#pragma unroll
        for (int p = 0; p < PT; ++p) {
          const double2 g = green<V>(tx[p], ty[p], tz[p], xs, ys, zs, tab);
          ar[p] = fma(g.x, qs.x, fma(-g.y, qs.y, ar[p]));
          ai[p] = fma(g.x, qs.y, fma(g.y, qs.x, ai[p]));
          if ((V & V_TWOACC) && (p & 1)) {
            cr2 = fma(g.x, tq[p].x, fma(-g.y, tq[p].y, cr2));
            ci2 = fma(g.x, tq[p].y, fma(g.y, tq[p].x, ci2));
          } else {
            cr = fma(g.x, tq[p].x, fma(-g.y, tq[p].y, cr));
            ci = fma(g.x, tq[p].y, fma(g.y, tq[p].x, ci));
          }
        }
        if (!(V & V_NOSHFL)) {
          cr = __shfl_sync(0xffffffffu, cr, (lane + 1) & 31);
          ci = __shfl_sync(0xffffffffu, ci, (lane + 1) & 31);
          if (V & V_TWOACC) {
            cr2 = __shfl_sync(0xffffffffu, cr2, (lane + 1) & 31);
            ci2 = __shfl_sync(0xffffffffu, ci2, (lane + 1) & 31);
          }
        }
      }
      col[warp][base + lane] = make_double2(cr + cr2, ci + ci2);
    }
    __syncthreads();
    double2 sum = col[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < TPB / 32; ++w) sum.x += col[w][threadIdx.x].x, sum.y += col[w][threadIdx.x].y;
    csum.x += sum.x, csum.y += sum.y;
  }
  double sr = csum.x, si = csum.y;
#pragma unroll
  for (int p = 0; p < PT; ++p) sr += ar[p], si += ai[p];
  out[(int64_t)blockIdx.x * TPB + threadIdx.x] = make_double2(sr, si);
}

__global__ void dfma3_loop(double *out, int iters, const double *in) {
  double a[8], b[8], x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = in[i] + threadIdx.x, b[i] = in[8 + i] - threadIdx.x, x[i] = in[16 + i];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(a[(i + u) & 7], b[(i + 3 * u) & 7], x[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

template <int V, int PT, int MINB, int UNR = 2>
static void run(const char *name, const double *ux, const double *uy, const double *uz, const double2 *q,
                double2 *out, int nitems, int ns, double mhz, int sms) {
  const int nt = PT * TPB;
  sym_kernel<V, PT, MINB, UNR><<<nitems, TPB>>>(ux, uy, uz, q, nt, ns, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    sym_kernel<V, PT, MINB, UNR><<<nitems, TPB>>>(ux, uy, uz, q, nt, ns, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, sym_kernel<V, PT, MINB, UNR>);
  const double evals = (double)nitems * nt * ns;
  printf("{\"variant\": \"%s\", \"regs\": %d, \"ms\": %.3f, \"gevals_per_s\": %.2f, "
         "\"fp64_ops_per_clk_sm_at_33\": %.2f}\n",
         name, fa.numRegs, best, evals / best / 1e6, 33.0 * evals / (best * 1e-3) / (sms * mhz * 1e6));
}

int main(int argc, char **argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int nitems = sms * 3 * 8, ns = 2048;
  const int64_t npts = (int64_t)nitems * 2048 + 7777 + 4096;
  std::vector<double> hx(npts), hy(npts), hz(npts);
  std::vector<double2> hq(npts);
  uint64_t st = 12345;
  auto rnd = [&]() { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return (double)(st >> 11) / 9007199254740992.0; };
  for (int64_t i = 0; i < npts; ++i) {
    hx[i] = 8192.0 * rnd(), hy[i] = 8192.0 * rnd(), hz[i] = 8192.0 * rnd();  // ~ C4 leaf pair span in table steps
    hq[i] = make_double2(rnd() - 0.5, rnd() - 0.5);
  }
  double *ux, *uy, *uz;
  double2 *q, *out;
  CK(cudaMalloc(&ux, npts * 8)); CK(cudaMalloc(&uy, npts * 8)); CK(cudaMalloc(&uz, npts * 8));
  CK(cudaMalloc(&q, npts * 16)); CK(cudaMalloc(&out, (int64_t)nitems * TPB * 16));
  CK(cudaMemcpy(ux, hx.data(), npts * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(uy, hy.data(), npts * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(uz, hz.data(), npts * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(q, hq.data(), npts * 16, cudaMemcpyHostToDevice));

  run<0, 4, 2>("base_pt4", ux, uy, uz, q, out, nitems, ns, mhz, sms);
  run<0, 4, 2, 1>("pt4_unr1", ux, uy, uz, q, out, nitems, ns, mhz, sms);
  run<0, 4, 2, 4>("pt4_unr4", ux, uy, uz, q, out, nitems, ns, mhz, sms);
  run<0, 8, 1>("pt8", ux, uy, uz, q, out, nitems / 2, ns, mhz, sms);
  run<0, 8, 1, 1>("pt8_unr1", ux, uy, uz, q, out, nitems / 2, ns, mhz, sms);
  run<0, 6, 1>("pt6", ux, uy, uz, q, out, nitems * 2 / 3, ns, mhz, sms);
  run<0, 6, 1, 1>("pt6_unr1", ux, uy, uz, q, out, nitems * 2 / 3, ns, mhz, sms);
  run<0, 5, 2, 1>("pt5_unr1", ux, uy, uz, q, out, nitems * 4 / 5, ns, mhz, sms);
  run<V_MACORD, 4, 2>("pt4_macord", ux, uy, uz, q, out, nitems, ns, mhz, sms);
  run<V_MACORD, 8, 1>("pt8_macord", ux, uy, uz, q, out, nitems / 2, ns, mhz, sms);
  run<V_NOTAB | V_NOSHFL, 8, 1>("pt8_notab_noshfl", ux, uy, uz, q, out, nitems / 2, ns, mhz, sms);
  {
    double *in, *o;
    CK(cudaMalloc(&in, 24 * 8)); CK(cudaMalloc(&o, 8));
    std::vector<double> hi(24);
    for (int i = 0; i < 24; ++i) hi[i] = 0.999 + 1e-4 * i;
    CK(cudaMemcpy(in, hi.data(), 24 * 8, cudaMemcpyHostToDevice));
    for (int occ : {3, 4, 8}) {
      const int blocks = sms * occ, threads = 128, iters = 20000;
      dfma3_loop<<<blocks, threads>>>(o, 100, in);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0), cudaEventCreate(&e1);
      cudaEventRecord(e0);
      dfma3_loop<<<blocks, threads>>>(o, iters, in);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double f = (double)blocks * threads * iters * 16 * 8;
      printf("{\"variant\": \"dfma3_regs\", \"warps_per_sm\": %d, \"ms\": %.3f, \"dfma_per_clk_sm\": %.2f}\n", occ * 4, ms,
             f / (ms * 1e-3) / (sms * mhz * 1e6));
    }
  }
  return 0;
}
