// M2L transfer pass and the GPU side of the precompute (product code, sm_100a).
//   M2L   I^l_a(s) = sum_{b in I(B_a)} M^l_b(s) T_{l, c_b - c_a}(s)
//   Alg.1 bandlimited modified transfer function T^{s,L}, one CTA per (offset, phi column)
//         (P:508-530); phi-truncation to T^{s,LL} when N_phi < 2 ell + 2
#include <cuda_runtime.h>
#include <cstdint>

#include "hfmm_impl.h"

namespace hfmm {

__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// ------------------------------------ M2L --------------------------------------------------
// grid: (k tiles, target boxes); thread per direction k; interaction list read by broadcast.
constexpr int M2L_TPB = 256;

__global__ void __launch_bounds__(M2L_TPB) m2l_kernel(int32_t box0, int64_t K, const int32_t *__restrict__ row,
                                                      const int32_t *__restrict__ src,
                                                      const int32_t *__restrict__ oid,
                                                      const double2 *__restrict__ T,
                                                      const double2 *__restrict__ M,
                                                      double2 *__restrict__ I) {
  const int32_t a = box0 + blockIdx.x;   // boxes on x (gridDim.y is limited to 65535)
  const int64_t k = (int64_t)blockIdx.y * M2L_TPB + threadIdx.x;
  if (k >= K) return;
  double2 acc = make_double2(0.0, 0.0);
  const int32_t e0 = row[a], e1 = row[a + 1];
  int32_t e = e0;
  for (; e + 1 < e1; e += 2) {  // two partners in flight
    const double2 t0 = __ldg(&T[(int64_t)oid[e] * K + k]);
    const double2 m0 = __ldg(&M[(int64_t)src[e] * K + k]);
    const double2 t1 = __ldg(&T[(int64_t)oid[e + 1] * K + k]);
    const double2 m1 = __ldg(&M[(int64_t)src[e + 1] * K + k]);
    acc = cfma(t0, m0, acc);
    acc = cfma(t1, m1, acc);
  }
  if (e < e1) acc = cfma(__ldg(&T[(int64_t)oid[e] * K + k]), __ldg(&M[(int64_t)src[e] * K + k]), acc);
  I[(int64_t)a * K + k] = acc;
}

void launch_m2l(int32_t box0, int32_t box1, int64_t K, const int32_t *row, const int32_t *src,
                const int32_t *oid, const double2 *T, const double2 *M, double2 *I, cudaStream_t s) {
  if (box1 <= box0 || K <= 0) return;
  dim3 grid((unsigned)(box1 - box0), (unsigned)((K + M2L_TPB - 1) / M2L_TPB));
  m2l_kernel<<<grid, M2L_TPB, 0, s>>>(box0, K, row, src, oid, T, M, I);
}

// M2L with the 34 canonical tables (NEXT 3): the table of interaction e is
// T[c_e][perm[op_e][k]], c_e / op_e packed in sym[e] = c << 4 | op (reflection / swap op).  The
// permuted reads are reversed runs of a row (reflections) and stay coalesced.
__global__ void __launch_bounds__(M2L_TPB) m2l_sym_kernel(int32_t box0, int64_t K, const int32_t *__restrict__ row,
                                                          const int32_t *__restrict__ src,
                                                          const int32_t *__restrict__ sym,
                                                          const int32_t *__restrict__ perm,
                                                          const double2 *__restrict__ T,
                                                          const double2 *__restrict__ M,
                                                          double2 *__restrict__ I) {
  const int32_t a = box0 + blockIdx.x;
  const int64_t k = (int64_t)blockIdx.y * M2L_TPB + threadIdx.x;
  if (k >= K) return;
  double2 acc = make_double2(0.0, 0.0);
  const int32_t e0 = row[a], e1 = row[a + 1];
  int32_t e = e0;
  for (; e + 1 < e1; e += 2) {  // two partners in flight
    const int32_t c0 = sym[e], c1 = sym[e + 1];
    const int32_t p0 = __ldg(&perm[(int64_t)(c0 & 15) * K + k]), p1 = __ldg(&perm[(int64_t)(c1 & 15) * K + k]);
    const double2 t0 = __ldg(&T[(int64_t)(c0 >> 4) * K + p0]);
    const double2 m0 = __ldg(&M[(int64_t)src[e] * K + k]);
    const double2 t1 = __ldg(&T[(int64_t)(c1 >> 4) * K + p1]);
    const double2 m1 = __ldg(&M[(int64_t)src[e + 1] * K + k]);
    acc = cfma(t0, m0, acc);
    acc = cfma(t1, m1, acc);
  }
  if (e < e1) {
    const int32_t c0 = sym[e];
    const int32_t p0 = __ldg(&perm[(int64_t)(c0 & 15) * K + k]);
    acc = cfma(__ldg(&T[(int64_t)(c0 >> 4) * K + p0]), __ldg(&M[(int64_t)src[e] * K + k]), acc);
  }
  I[(int64_t)a * K + k] = acc;
}

void launch_m2l_sym(int32_t box0, int32_t box1, int64_t K, const int32_t *row, const int32_t *src,
                    const int32_t *sym, const int32_t *perm, const double2 *T, const double2 *M, double2 *I,
                    cudaStream_t s) {
  if (box1 <= box0 || K <= 0) return;
  dim3 grid((unsigned)(box1 - box0), (unsigned)((K + M2L_TPB - 1) / M2L_TPB));
  m2l_sym_kernel<<<grid, M2L_TPB, 0, s>>>(box0, K, row, src, sym, perm, T, M, I);
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

}  // namespace hfmm
