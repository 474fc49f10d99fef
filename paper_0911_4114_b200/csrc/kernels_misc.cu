// GPU side of the precompute (product code, sm_100a); the M2L pass is in kernels_m2l.cu.
//   Alg.1 bandlimited modified transfer function T^{s,L}, one CTA per (offset, phi column)
//         (P:508-530); phi-truncation to T^{s,LL} when N_phi < 2 ell + 2
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "hfmm_impl.h"

namespace hfmm {

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// ------------------------------------ Alg. 1 -----------------------------------------------
// One CTA per (phi column q, offset o).  shared: c_n, samples, spectrum, truncated spectrum,
// twiddles of length P = 2 ell + 1 and N_theta.
constexpr int ALG1_TPB = 256;

__device__ __forceinline__ double sin_spec(int n) {  // F_n[|sin theta|]
  return (n & 1) ? 0.0 : 2.0 / (3.14159265358979323846 * (1.0 - (double)n * (double)n));
}

__global__ void __launch_bounds__(ALG1_TPB) alg1_kernel(const double2 *__restrict__ coef,
                                                        const int32_t *__restrict__ coef_of_offset,
                                                        const double *__restrict__ r0hat, int ell, int nth,
                                                        int nphf, int qcount, double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int P = 2 * ell + 1;
  const int nb = nth / 2 - 1;
  double2 *c = sm;                 // ell + 1
  double2 *samp = c + (ell + 1);   // P
  double2 *tt = samp + P;          // P  (freq -ell..ell)
  double2 *ts = tt + P;            // 2 nb + 1
  double2 *twP = ts + (2 * nb + 1);// P   e^{-2 pi i t / P}
  double2 *twN = twP + P;          // nth e^{+2 pi i t / nth}
  const int q = blockIdx.x, o = blockIdx.y;
  const double2 *cg = coef + (int64_t)coef_of_offset[o] * (ell + 1);
  for (int n = threadIdx.x; n <= ell; n += blockDim.x) c[n] = cg[n];
  for (int t = threadIdx.x; t < P; t += blockDim.x) {
    double s, cs;
    sincospi(-2.0 * (double)t / (double)P, &s, &cs);
    twP[t] = make_double2(cs, s);
  }
  for (int t = threadIdx.x; t < nth; t += blockDim.x) {
    double s, cs;
    sincospi(2.0 * (double)t / (double)nth, &s, &cs);
    twN[t] = make_double2(cs, s);
  }
  __syncthreads();
  double sp, cp;
  sincospi(2.0 * (double)q / (double)nphf, &sp, &cp);
  const double rx = r0hat[3 * o], ry = r0hat[3 * o + 1], rz = r0hat[3 * o + 2];
  // step 1: (1/2) T_{ell, r0}(theta_j, phi_q), theta_j = 2 pi j / P   (Alg. 1 line 3)
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    double st, ct;
    sincospi(2.0 * (double)j / (double)P, &st, &ct);
    double t = fma(cp * st, rx, fma(sp * st, ry, ct * rz));
    t = fmin(1.0, fmax(-1.0, t));
    double p0 = 1.0, p1 = t;
    double2 acc = c[0];
    if (ell >= 1) acc = make_double2(fma(c[1].x, p1, acc.x), fma(c[1].y, p1, acc.y));
    for (int n = 1; n < ell; ++n) {
      const double p2 = (fma((double)(2 * n + 1) * t, p1, -(double)n * p0)) / (double)(n + 1);
      acc = make_double2(fma(c[n + 1].x, p2, acc.x), fma(c[n + 1].y, p2, acc.y));
      p0 = p1;
      p1 = p2;
    }
    samp[j] = make_double2(0.5 * acc.x, 0.5 * acc.y);
  }
  __syncthreads();
  // step 2: spectrum T~_f, |f| <= ell  (Alg. 1 line 4)
  for (int f = threadIdx.x - ell; f <= ell; f += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const int fm = (f % P + P) % P;
    int idx = 0;
    for (int j = 0; j < P; ++j) {
      acc = cfma(samp[j], twP[idx], acc);
      idx += fm;
      if (idx >= P) idx -= P;
    }
    tt[f + ell] = make_double2(acc.x / P, acc.y / P);
  }
  __syncthreads();
  // step 3: convolution with F[|sin|], truncated to |n| <= N_theta/2 - 1  (Alg. 1 lines 5-6)
  for (int n = threadIdx.x - nb; n <= nb; n += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int f = -ell; f <= ell; ++f) {
      const double w = sin_spec(n - f);
      acc = make_double2(fma(tt[f + ell].x, w, acc.x), fma(tt[f + ell].y, w, acc.y));
    }
    ts[n + nb] = acc;
  }
  __syncthreads();
  // step 4: inverse transform at theta_p = 2 pi p / N_theta  (Alg. 1 line 7)
  for (int p = threadIdx.x; p < nth; p += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    int idx = ((-nb * p) % nth + nth) % nth;
    for (int n = -nb; n <= nb; ++n) {
      acc = cfma(ts[n + nb], twN[idx], acc);
      idx += p;
      if (idx >= nth) idx -= nth;
    }
    out[((int64_t)o * nth + p) * qcount + q] = acc;
  }
}

void launch_alg1_tables(const double2 *coef, const int32_t *coef_of_offset, const double *r0hat, int noff,
                        int ell, int nth, int nphf, int qcount, double2 *out, cudaStream_t s) {
  const int P = 2 * ell + 1;
  size_t smem = sizeof(double2) * ((size_t)(ell + 1) + 3 * (size_t)P + (size_t)(nth - 1) + (size_t)nth);
  cudaFuncSetAttribute((const void *)alg1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)qcount, (unsigned)noff);
  alg1_kernel<<<grid, ALG1_TPB, smem, s>>>(coef, coef_of_offset, r0hat, ell, nth, nphf, qcount, out);
}

// phi-truncation of each full row (length nphf) to |m| <= nph/2 - 1, sampled at m < nph/2
__global__ void phi_anterp_kernel(const double2 *__restrict__ full, int nth, int nphf, int nph,
                                  double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int64_t rowid = blockIdx.x;  // o * nth + p
  const double2 *row = full + rowid * nphf;
  const int K = (nph - 1) / 2 < (nphf - 1) / 2 ? (nph - 1) / 2 : (nphf - 1) / 2;
  double2 *spec = sm;  // 2K + 1
  for (int f = threadIdx.x - K; f <= K; f += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int q = 0; q < nphf; ++q) {
      double s, c;
      const int e = (int)(((int64_t)f * q % nphf + nphf) % nphf);
      sincospi(-2.0 * (double)e / (double)nphf, &s, &c);
      acc = cfma(row[q], make_double2(c, s), acc);
    }
    spec[f + K] = make_double2(acc.x / nphf, acc.y / nphf);
  }
  __syncthreads();
  for (int m = threadIdx.x; m < nph / 2; m += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int f = -K; f <= K; ++f) {
      double s, c;
      const int e = (int)(((int64_t)f * m % nph + nph) % nph);
      sincospi(2.0 * (double)e / (double)nph, &s, &c);
      acc = cfma(spec[f + K], make_double2(c, s), acc);
    }
    out[rowid * (nph / 2) + m] = acc;
  }
}

void launch_phi_anterp(const double2 *full, int noff, int nth, int nphf, int nph, double2 *out, cudaStream_t s) {
  size_t smem = sizeof(double2) * (size_t)nph;
  phi_anterp_kernel<<<(unsigned)(noff * nth), 128, smem, s>>>(full, nth, nphf, nph, out);
}

__global__ void absmax_kernel(const double2 *__restrict__ v, int64_t n, unsigned long long *out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, hypot(v[i].x, v[i].y));
  for (int off = 16; off; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

void launch_absmax(const double2 *v, int64_t n, double *out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  absmax_kernel<<<148 * 4, 256, 0, s>>>(v, n, reinterpret_cast<unsigned long long *>(out));
}

// M2L halo pack / scatter: one CTA row per box (blockIdx.y strided), lanes over k (coalesced)
__global__ void gather_boxes_kernel(const double2 *__restrict__ in, const int64_t *__restrict__ iidx,
                                    double2 *__restrict__ out, const int64_t *__restrict__ oidx, int64_t count,
                                    int64_t K) {
  for (int64_t i = blockIdx.y; i < count; i += gridDim.y) {
    const double2 *src = in + (iidx ? iidx[i] : i) * K;
    double2 *dst = out + (oidx ? oidx[i] : i) * K;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x)
      dst[k] = src[k];
  }
}

void launch_gather_boxes(const double2 *in, const int64_t *iidx, double2 *out, const int64_t *oidx, int64_t count,
                         int64_t K, cudaStream_t s) {
  if (count <= 0 || K <= 0) return;
  const unsigned gx = (unsigned)std::min<int64_t>((K + 255) / 256, 64);
  const unsigned gy = (unsigned)std::min<int64_t>(count, 65535);
  gather_boxes_kernel<<<dim3(gx, gy), 256, 0, s>>>(in, iidx, out, oidx, count, K);
}

}  // namespace hfmm
