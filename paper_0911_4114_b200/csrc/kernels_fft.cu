// Fourier interpolation / anterpolation on the sphere (product code, sm_100a).
//   P:373-378  interpolation = zero-pad the Fourier coefficients, anterpolation = truncate
//   P:512      kept band |k| <= min(N, N')/2 - 1 (Nyquist dropped; R-6)
//   P:724-749  5-step 2-D procedure between quadratures, with eqn:NumSphereSym
//              used to build theta-periodic columns / full phi-rows from half storage.
// Each 1-D resample N -> N' is: forward FFT (length N), spectral pad/truncate with 1/N,
// inverse FFT (length N') computed as conj(FFT(conj(.))).  FFTs are mixed-radix Stockham
// (radices 4, 2, 3, 5, 7; autosort, ping-pong buffers) run by one warp per sequence in
// shared memory, with exact twiddles e^{-2 pi i t/N} from a per-length table in global
// memory (read through L1).
//
// The two-pass layout (rows pass, columns pass, intermediate in global memory / L2):
//   upward   (M2M): rows n <= N_theta/2 resampled N_phi -> N'_phi (step 1), then
//            columns m < N'_phi/2 (step 2) resampled N_theta -> N'_theta (step 3), multiplied by
//            the translation e^{i kappa s.(c_child - c_parent)} and accumulated over the 8
//            children; steps 4-5 are the identity for interpolation (the phi band already fits).
//   downward (L2L): columns of conj(shift) * L_parent (steps 1-2 are the identity for
//            anterpolation) resampled N_theta -> N'_theta (step 3), then rows n <= N'_theta/2
//            rebuilt (step 4) and resampled N_phi -> N'_phi (step 5), + I_child.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "hfmm_impl.h"

namespace hfmm {

struct FFTLen {
  int N;
  int nr;
  int radix[12];
  const double2 *tw;  // e^{-2 pi i t/N}, t < N
};

static FFTLen make_len(const TwiddleSet &ts, int N) {
  FFTLen L;
  L.N = N;
  L.nr = 0;
  int m = N;
  for (int r : {4, 2, 3, 5, 7})
    while (m % r == 0) {
      L.radix[L.nr++] = r;
      m /= r;
    }
  L.tw = (N < 1024 && ts.offset[N] >= 0) ? ts.d + ts.offset[N] : nullptr;
  return L;
}

void TwiddleSet::build(const std::vector<int> &lengths) {
  for (int i = 0; i < 1024; ++i) offset[i] = -1;
  std::vector<double2> h;
  for (int N : lengths) {
    if (N <= 0 || N >= 1024 || offset[N] >= 0) continue;
    offset[N] = (int)h.size();
    for (int t = 0; t < N; ++t) {
      long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)t / (long double)N;
      h.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
    }
  }
  if (d) cudaFree(d);
  d = nullptr;
  if (!h.empty()) {
    cudaMalloc(&d, h.size() * sizeof(double2));
    cudaMemcpy(d, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
  }
}

void TwiddleSet::free_all() {
  if (d) cudaFree(d);
  d = nullptr;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// forward small DFTs, out[t] = sum_s v[s] e^{-2 pi i s t / R}
__device__ __forceinline__ void bfly2(double2 *v) {
  double2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
__device__ __forceinline__ void bfly4(double2 *v) {
  double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  double2 b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
  // multiply b1 by -i
  double2 b1m = make_double2(b1.y, -b1.x);
  v[0] = cadd(a0, b0);
  v[2] = csub(a0, b0);
  v[1] = cadd(a1, b1m);
  v[3] = csub(a1, b1m);
}
__device__ __forceinline__ void bfly3(double2 *v) {
  const double c = -0.5, s = -0.86602540378443864676372317075294;  // e^{-2 pi i/3}
  double2 t1 = cadd(v[1], v[2]), t2 = csub(v[1], v[2]);
  double2 m1 = make_double2(fma(c, t1.x, v[0].x), fma(c, t1.y, v[0].y));
  double2 m2 = make_double2(-s * t2.y, s * t2.x);  // i s t2
  v[0] = cadd(v[0], t1);
  v[1] = cadd(m1, m2);
  v[2] = csub(m1, m2);
}
// e^{-2 pi i e / R} for R = 5, 7 (compile-time constants after unrolling)
template <int R>
__device__ __forceinline__ void bfly_generic(double2 *v) {
  const double c5[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410, -0.80901699437494742410,
                        0.30901699437494742410};
  const double s5[5] = {0.0, -0.95105651629515357212, -0.58778525229247312917, 0.58778525229247312917,
                        0.95105651629515357212};
  const double c7[7] = {1.0, 0.62348980185873353053, -0.22252093395631440429, -0.90096886790241912624,
                        -0.90096886790241912624, -0.22252093395631440429, 0.62348980185873353053};
  const double s7[7] = {0.0, -0.78183148246802980871, -0.97492791218182360702, -0.43388373911755812048,
                        0.43388373911755812048, 0.97492791218182360702, 0.78183148246802980871};
  double2 o[R];
#pragma unroll
  for (int t = 0; t < R; ++t) {
    double2 acc = v[0];
#pragma unroll
    for (int s = 1; s < R; ++s) {
      const int e = (s * t) % R;
      const double cs = (R == 5) ? c5[e] : c7[e];
      const double sn = (R == 5) ? s5[e] : s7[e];
      acc = make_double2(fma(v[s].x, cs, fma(-v[s].y, sn, acc.x)), fma(v[s].x, sn, fma(v[s].y, cs, acc.y)));
    }
    o[t] = acc;
  }
#pragma unroll
  for (int t = 0; t < R; ++t) v[t] = o[t];
}

template <int R>
__device__ __forceinline__ void stockham_stage(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                               int N, int Ns, const double2 *__restrict__ tw, int lane) {
  const int stride = N / R;
  const int tstep = N / (Ns * R);
  for (int j = lane; j < stride; j += 32) {
    const int k = j % Ns;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v[r] = src[j + r * stride];
      if (r) v[r] = cmul(v[r], __ldg(&tw[k * r * tstep]));
    }
    if (R == 2) bfly2(v);
    else if (R == 4) bfly4(v);
    else if (R == 3) bfly3(v);
    else bfly_generic<R>(v);
    const int idxD = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[idxD + r * Ns] = v[r];
  }
  __syncwarp();
}

// forward FFT of a[0..N) (warp-cooperative); returns the buffer holding the result (a or b)
__device__ double2 *warp_fft(double2 *a, double2 *b, const FFTLen &L, int lane) {
  double2 *src = a, *dst = b;
  int Ns = 1;
  for (int s = 0; s < L.nr; ++s) {
    const int R = L.radix[s];
    switch (R) {
      case 4: stockham_stage<4>(src, dst, L.N, Ns, L.tw, lane); break;
      case 2: stockham_stage<2>(src, dst, L.N, Ns, L.tw, lane); break;
      case 3: stockham_stage<3>(src, dst, L.N, Ns, L.tw, lane); break;
      case 5: stockham_stage<5>(src, dst, L.N, Ns, L.tw, lane); break;
      default: stockham_stage<7>(src, dst, L.N, Ns, L.tw, lane); break;
    }
    double2 *t = src;
    src = dst;
    dst = t;
    Ns *= R;
  }
  return src;
}

// 1-D Fourier resample of A[0..N) to length N'; returns Z with y[t] = conj(Z[t]).
__device__ double2 *warp_resample(double2 *A, double2 *B, const FFTLen &Lin, const FFTLen &Lout, int lane) {
  double2 *X = warp_fft(A, B, Lin, lane);
  double2 *Y = (X == A) ? B : A;
  const int N = Lin.N, Np = Lout.N;
  const int K = (min(N, Np) - 1) / 2;
  const double sc = 1.0 / (double)N;
  for (int t = lane; t < Np; t += 32) {
    const int f = (t <= Np / 2) ? t : t - Np;
    double2 v = make_double2(0.0, 0.0);
    if (f <= K && f >= -K) {
      const double2 x = X[f >= 0 ? f : f + N];
      v = make_double2(x.x * sc, -x.y * sc);  // conj for the inverse transform
    }
    Y[t] = v;
  }
  __syncwarp();
  return warp_fft(Y, X, Lout, lane);
}

constexpr int FFT_WARPS = 4;

// ------------------------------- upward: rows pass -----------------------------------------
__global__ void __launch_bounds__(32 * FFT_WARPS) rows_up_kernel(const double2 *__restrict__ in, int64_t nbox,
                                                                 int nth, int nph, FFTLen Lin, FFTLen Lout,
                                                                 double2 *__restrict__ tmp) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int maxn = max(Lin.N, Lout.N);
  double2 *A = sm + (size_t)warp * 2 * maxn, *B = A + maxn;
  const int rows = nth / 2 + 1;
  const int64_t seq = (int64_t)blockIdx.x * FFT_WARPS + warp;
  if (seq >= nbox * rows) return;
  const int64_t b = seq / rows;
  const int n = (int)(seq % rows);
  const int h = nph / 2;
  const double2 *r0 = in + ((int64_t)b * nth + n) * h;
  const double2 *r1 = in + ((int64_t)b * nth + (nth - n) % nth) * h;
  for (int m = lane; m < nph; m += 32) A[m] = (m < h) ? r0[m] : r1[m - h];
  __syncwarp();
  double2 *Z = warp_resample(A, B, Lin, Lout, lane);
  double2 *o = tmp + ((int64_t)b * rows + n) * Lout.N;
  for (int t = lane; t < Lout.N; t += 32) o[t] = conjd(Z[t]);
}

// ------------------------------- upward: columns pass (+ shift, accumulate) -----------------
__global__ void __launch_bounds__(32 * FFT_WARPS) cols_up_kernel(const double2 *__restrict__ tmp, int nth, int nph2,
                                                                 const int32_t *__restrict__ cbeg, int64_t cbase,
                                                                 const int8_t *__restrict__ oct, int64_t nparent,
                                                                 const double2 *__restrict__ shift,
                                                                 FFTLen Lin, FFTLen Lout,
                                                                 double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int maxn = max(Lin.N, Lout.N);
  double2 *A = sm + (size_t)warp * 3 * maxn, *B = A + maxn, *C = B + maxn;
  const int h2 = nph2 / 2;
  const int64_t seq = (int64_t)blockIdx.x * FFT_WARPS + warp;
  if (seq >= nparent * h2) return;
  const int64_t p = seq / h2;
  const int m = (int)(seq % h2);
  const int rows = nth / 2 + 1;
  const int nth2 = Lout.N;
  for (int t = lane; t < nth2; t += 32) C[t] = make_double2(0.0, 0.0);
  const int64_t c0 = cbeg ? cbeg[p] : p, c1 = cbeg ? cbeg[p + 1] : p + 1;
  for (int64_t c = c0; c < c1; ++c) {
    const double2 *tc = tmp + (int64_t)(c - cbase) * rows * nph2;
    for (int n = lane; n < nth; n += 32)
      A[n] = (2 * n <= nth) ? tc[(int64_t)n * nph2 + m] : tc[(int64_t)(nth - n) * nph2 + m + h2];
    __syncwarp();
    double2 *Z = warp_resample(A, B, Lin, Lout, lane);
    const double2 *sh = shift ? shift + (int64_t)(oct ? oct[c] : 0) * nth2 * h2 : nullptr;
    for (int t = lane; t < nth2; t += 32) {
      double2 v = conjd(Z[t]);
      if (sh) v = cmul(v, sh[(int64_t)t * h2 + m]);
      C[t] = cadd(C[t], v);
    }
    __syncwarp();
  }
  double2 *o = out + (int64_t)p * nth2 * h2;
  for (int t = lane; t < nth2; t += 32) o[(int64_t)t * h2 + m] = C[t];
}

// ------------------------------- downward: columns pass ------------------------------------
__global__ void __launch_bounds__(32 * FFT_WARPS) cols_down_kernel(const double2 *__restrict__ in, int nph,
                                                                   const int32_t *__restrict__ par,
                                                                   const int8_t *__restrict__ oct, int64_t nchild,
                                                                   const double2 *__restrict__ shift,
                                                                   FFTLen Lin, FFTLen Lout,
                                                                   double2 *__restrict__ tmp) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int maxn = max(Lin.N, Lout.N);
  double2 *A = sm + (size_t)warp * 2 * maxn, *B = A + maxn;
  const int h = nph / 2;
  const int64_t seq = (int64_t)blockIdx.x * FFT_WARPS + warp;
  if (seq >= nchild * h) return;
  const int64_t c = seq / h;
  const int m = (int)(seq % h);
  const int64_t p = par ? par[c] : c;
  const int nth = Lin.N, nth2 = Lout.N;
  const double2 *src = in + (int64_t)p * nth * h;
  const double2 *sh = shift ? shift + (int64_t)(oct ? oct[c] : 0) * nth * h : nullptr;
  for (int n = lane; n < nth; n += 32) {
    double2 v = src[(int64_t)n * h + m];
    if (sh) v = cmul(v, conjd(sh[(int64_t)n * h + m]));  // e^{i kappa s.(c_parent - c_child)}
    A[n] = v;
  }
  __syncwarp();
  double2 *Z = warp_resample(A, B, Lin, Lout, lane);
  double2 *o = tmp + (int64_t)c * nth2 * h;
  for (int t = lane; t < nth2; t += 32) o[(int64_t)t * h + m] = conjd(Z[t]);
}

// ------------------------------- downward: rows pass (+ add) -------------------------------
__global__ void __launch_bounds__(32 * FFT_WARPS) rows_down_kernel(const double2 *__restrict__ tmp, int64_t nbox,
                                                                   int nth2, int nph, FFTLen Lin, FFTLen Lout,
                                                                   const double2 *__restrict__ add,
                                                                   double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int maxn = max(Lin.N, Lout.N);
  double2 *A = sm + (size_t)warp * 2 * maxn, *B = A + maxn;
  const int rows = nth2 / 2 + 1;
  const int64_t seq = (int64_t)blockIdx.x * FFT_WARPS + warp;
  if (seq >= nbox * rows) return;
  const int64_t c = seq / rows;
  const int n = (int)(seq % rows);
  const int h = nph / 2, h2 = Lout.N / 2;
  const double2 *r0 = tmp + ((int64_t)c * nth2 + n) * h;
  const double2 *r1 = tmp + ((int64_t)c * nth2 + (nth2 - n) % nth2) * h;
  for (int m = lane; m < nph; m += 32) A[m] = (m < h) ? r0[m] : r1[m - h];
  __syncwarp();
  double2 *Z = warp_resample(A, B, Lin, Lout, lane);
  const int64_t o0 = ((int64_t)c * nth2 + n) * h2;
  for (int t = lane; t < h2; t += 32) {
    double2 v = conjd(Z[t]);
    if (add) v = cadd(v, add[o0 + t]);
    out[o0 + t] = v;
  }
  if (n > 0 && 2 * n < nth2) {
    const int64_t o1 = ((int64_t)c * nth2 + (nth2 - n)) * h2;
    for (int t = lane; t < h2; t += 32) {
      double2 v = conjd(Z[t + h2]);
      if (add) v = cadd(v, add[o1 + t]);
      out[o1 + t] = v;
    }
  }
}

static unsigned nblocks(int64_t seqs) { return (unsigned)((seqs + FFT_WARPS - 1) / FFT_WARPS); }

static void set_smem(const void *fn, size_t bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_rows_up(const double2 *in, int64_t nbox, int nth, int nph, int nph2, double2 *tmp,
                    const TwiddleSet &tw, cudaStream_t s) {
  FFTLen Li = make_len(tw, nph), Lo = make_len(tw, nph2);
  size_t smem = (size_t)FFT_WARPS * 2 * std::max(nph, nph2) * sizeof(double2);
  set_smem((const void *)rows_up_kernel, smem);
  int64_t seqs = nbox * (nth / 2 + 1);
  if (seqs) rows_up_kernel<<<nblocks(seqs), 32 * FFT_WARPS, smem, s>>>(in, nbox, nth, nph, Li, Lo, tmp);
}

void launch_cols_up(const double2 *tmp, int nth, int nph2, int nth2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, int64_t nparent, const double2 *shift, double2 *out,
                    const TwiddleSet &tw, cudaStream_t s) {
  FFTLen Li = make_len(tw, nth), Lo = make_len(tw, nth2);
  size_t smem = (size_t)FFT_WARPS * 3 * std::max(nth, nth2) * sizeof(double2);
  set_smem((const void *)cols_up_kernel, smem);
  int64_t seqs = nparent * (nph2 / 2);
  if (seqs) cols_up_kernel<<<nblocks(seqs), 32 * FFT_WARPS, smem, s>>>(tmp, nth, nph2, cbeg, cbase, oct, nparent, shift, Li, Lo, out);
}

void launch_cols_down(const double2 *in, int nth, int nph, int nth2, const int32_t *par,
                      const int8_t *oct, int64_t nchild, const double2 *shift, double2 *tmp,
                      const TwiddleSet &tw, cudaStream_t s) {
  FFTLen Li = make_len(tw, nth), Lo = make_len(tw, nth2);
  size_t smem = (size_t)FFT_WARPS * 2 * std::max(nth, nth2) * sizeof(double2);
  set_smem((const void *)cols_down_kernel, smem);
  int64_t seqs = nchild * (nph / 2);
  if (seqs) cols_down_kernel<<<nblocks(seqs), 32 * FFT_WARPS, smem, s>>>(in, nph, par, oct, nchild, shift, Li, Lo, tmp);
}

void launch_rows_down(const double2 *tmp, int64_t nbox, int nth2, int nph, int nph2,
                      const double2 *add, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  FFTLen Li = make_len(tw, nph), Lo = make_len(tw, nph2);
  size_t smem = (size_t)FFT_WARPS * 2 * std::max(nph, nph2) * sizeof(double2);
  set_smem((const void *)rows_down_kernel, smem);
  int64_t seqs = nbox * (nth2 / 2 + 1);
  if (seqs) rows_down_kernel<<<nblocks(seqs), 32 * FFT_WARPS, smem, s>>>(tmp, nbox, nth2, nph, Li, Lo, add, out);
}

}  // namespace hfmm
