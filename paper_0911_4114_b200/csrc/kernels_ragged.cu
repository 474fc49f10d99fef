// Ragged quadrature support (R-15; Alg. 3 per row),
// product code, sm_100a.  A ragged level stores N_phi(theta_n)/2 points on row n (row offsets
// off[n]); the 5-step resample between a ragged grid and the rectangular calN_phi
// used by the two-pass FFT kernels is a per-row Fourier resample (step 1: N_phi(theta_n) ->
// calN_phi; step 5: calN_phi -> N_phi(theta_n)), band |f| <= (min(N, N') - 1)/2 (R-6).  Rows
// have individual lengths, so each CTA resamples one full row (built with eqn:NumSphereSym from
// the stored rows n and N_theta - n) by direct DFT sums over exact twiddle tables; these passes
// are a small part of the matvec.
#include <cuda_runtime.h>
#include <cstdint>
#include <map>

#include "hfmm_impl.h"

namespace hfmm {

constexpr int RG_TPB = 128;

__device__ __forceinline__ double2 rg_cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// spectrum of the full row x[0..N) on |f| <= K, times 1/N: spec[f + K]
__device__ void row_spectrum(const double2 *x, int N, int K, const double2 *__restrict__ twN, double2 *spec) {
  for (int f = (int)threadIdx.x - K; f <= K; f += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const int ff = f >= 0 ? f : f + N;
    int idx = 0;
    for (int j = 0; j < N; ++j) {  // e^{-2 pi i f j / N} = twN[(f j) mod N]
      const double2 w = __ldg(&twN[idx]);
      acc = make_double2(fma(x[j].x, w.x, fma(-x[j].y, w.y, acc.x)), fma(x[j].x, w.y, fma(x[j].y, w.x, acc.y)));
      idx += ff;
      if (idx >= N) idx -= N;
    }
    spec[f + K] = make_double2(acc.x / N, acc.y / N);
  }
}

// value at point t of a length-N2 row with spectrum spec (|f| <= K): sum_f spec e^{+2 pi i f t / N2}
__device__ __forceinline__ double2 row_eval(const double2 *spec, int K, int N2, int t,
                                            const double2 *__restrict__ twN2) {
  double2 acc = make_double2(0.0, 0.0);
  const long long tt = t;
  for (int f = -K; f <= K; ++f) {
    long long e = (tt * f) % N2;
    if (e < 0) e += N2;
    const double2 w = __ldg(&twN2[e]);  // e^{-2 pi i e / N2}; conjugate for the inverse
    const double2 s = spec[f + K];
    acc = make_double2(fma(s.x, w.x, fma(s.y, w.y, acc.x)), fma(s.y, w.x, fma(-s.x, w.y, acc.y)));
  }
  return acc;
}

// ---- tables: rectangular T^{s,LL} [NC][nth][nphr/2] -> ragged [NC][K] (rows truncated to
// |m| <= N_phi(theta_n)/2 - 1 and sampled at 2 pi q / N_phi(theta_n)) -------------------
__global__ void __launch_bounds__(RG_TPB) ragged_tables_kernel(const double2 *__restrict__ Trect, int nth, int nphr,
                                                               const int32_t *__restrict__ rows,
                                                               const int64_t *__restrict__ off, int64_t K,
                                                               const double2 *__restrict__ tw_base,
                                                               const int32_t *__restrict__ tw_off,
                                                               double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int n = blockIdx.x, c = blockIdx.y;
  const int hr = nphr / 2, L = rows[n];
  double2 *x = sm, *spec = sm + nphr;
  const double2 *T = Trect + (int64_t)c * nth * hr;
  for (int j = threadIdx.x; j < nphr; j += blockDim.x)
    x[j] = j < hr ? T[(int64_t)n * hr + j] : T[(int64_t)((nth - n) % nth) * hr + j - hr];
  __syncthreads();
  const int Kb = (min(nphr, L) - 1) / 2;
  row_spectrum(x, nphr, Kb, tw_base + tw_off[nphr], spec);
  __syncthreads();
  for (int m = threadIdx.x; m < L / 2; m += blockDim.x)
    out[(int64_t)c * K + off[n] + m] = row_eval(spec, Kb, L, m, tw_base + tw_off[L]);
}

// ---- step 1: ragged rows -> rectangular half [nth][nphr/2] -----------------------------------------
// item o: input box in_box = par ? par[o] : o; optional pre-multiply by conj(shift[oct[o]][k]) on
// the input (ragged) grid; output box o.
__global__ void __launch_bounds__(RG_TPB) rag2rect_kernel(const double2 *__restrict__ in, int64_t in_K, int nth,
                                                          const int32_t *__restrict__ rows,
                                                          const int64_t *__restrict__ off,
                                                          const int32_t *__restrict__ par,
                                                          const int8_t *__restrict__ oct,
                                                          const double2 *__restrict__ shift, int nphr,
                                                          const double2 *__restrict__ tw_base,
                                                          const int32_t *__restrict__ tw_off,
                                                          double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int64_t o = blockIdx.x;
  const int n = blockIdx.y;  // n <= nth/2
  const int L = rows[n], h = L / 2, hr = nphr / 2;
  const int n2 = (nth - n) % nth;
  double2 *x = sm, *spec = sm + L;
  const int64_t ib = par ? par[o] : o;
  const double2 *src = in + ib * in_K;
  const double2 *sh = shift ? shift + (int64_t)(oct ? oct[o] : 0) * in_K : nullptr;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const int64_t k = j < h ? off[n] + j : off[n2] + j - h;
    double2 v = src[k];
    if (sh) {
      const double2 s = sh[k];
      v = rg_cmul(v, make_double2(s.x, -s.y));  // e^{i kappa s.(c_parent - c_child)}
    }
    x[j] = v;
  }
  __syncthreads();
  const int Kb = (min(L, nphr) - 1) / 2;
  row_spectrum(x, L, Kb, tw_base + tw_off[L], spec);
  __syncthreads();
  double2 *dst = out + o * (int64_t)nth * hr;
  for (int t = threadIdx.x; t < nphr; t += blockDim.x) {
    if (t >= hr && (n == 0 || 2 * n == nth)) continue;  // both halves are the same points
    const double2 v = row_eval(spec, Kb, nphr, t, tw_base + tw_off[nphr]);
    if (t < hr) dst[(int64_t)n * hr + t] = v;
    else dst[(int64_t)n2 * hr + t - hr] = v;
  }
}

// ---- step 5: rectangular half [nth][nphr/2] -> ragged rows --------------------------------------------
// item o: children c in [cbeg[o], cbeg[o+1]) (input row c - cbase) or c = o; each child's row is
// resampled to N_phi(theta_n), multiplied by shift[oct[c]][k] (ragged output grid) if shift, and
// summed; + add[o][k] if add.
__global__ void __launch_bounds__(RG_TPB) rect2rag_kernel(const double2 *__restrict__ in, int nth, int nphr,
                                                          const int32_t *__restrict__ cbeg, int64_t cbase,
                                                          const int8_t *__restrict__ oct,
                                                          const double2 *__restrict__ shift,
                                                          const double2 *__restrict__ add,
                                                          const int32_t *__restrict__ rows,
                                                          const int64_t *__restrict__ off, int64_t K,
                                                          const double2 *__restrict__ tw_base,
                                                          const int32_t *__restrict__ tw_off,
                                                          double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int64_t o = blockIdx.x;
  const int n = blockIdx.y;
  const int L = rows[n], h = L / 2, hr = nphr / 2;
  const int n2 = (nth - n) % nth;
  double2 *x = sm, *spec = sm + nphr, *acc = spec + nphr;
  const int64_t c0 = cbeg ? cbeg[o] : o, c1 = cbeg ? cbeg[o + 1] : o + 1;
  const int Kb = (min(L, nphr) - 1) / 2;
  for (int j = threadIdx.x; j < L; j += blockDim.x) acc[j] = make_double2(0.0, 0.0);
  for (int64_t c = c0; c < c1; ++c) {
    __syncthreads();
    const double2 *src = in + (c - cbase) * (int64_t)nth * hr;
    for (int j = threadIdx.x; j < nphr; j += blockDim.x)
      x[j] = j < hr ? src[(int64_t)n * hr + j] : src[(int64_t)n2 * hr + j - hr];
    __syncthreads();
    row_spectrum(x, nphr, Kb, tw_base + tw_off[nphr], spec);
    __syncthreads();
    const double2 *sh = shift ? shift + (int64_t)(oct ? oct[c] : 0) * K : nullptr;
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
      double2 v = row_eval(spec, Kb, L, t, tw_base + tw_off[L]);
      if (sh) v = rg_cmul(v, sh[t < h ? off[n] + t : off[n2] + t - h]);
      acc[t] = make_double2(acc[t].x + v.x, acc[t].y + v.y);
    }
  }
  __syncthreads();
  double2 *dst = out + o * K;
  const double2 *ad = add ? add + o * K : nullptr;
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    if (t >= h && (n == 0 || 2 * n == nth)) continue;
    const int64_t k = t < h ? off[n] + t : off[n2] + t - h;
    double2 v = acc[t];
    if (ad) v = make_double2(v.x + ad[k].x, v.y + ad[k].y);
    dst[k] = v;
  }
}

static const int32_t *twiddle_offsets_device(const TwiddleSet &tw) {
  // device copy of TwiddleSet::offset (lengths < kMaxFFT), one per TwiddleSet (one set per device)
  std::lock_guard<std::recursive_mutex> lk(cache_mutex());
  static std::map<const TwiddleSet *, int32_t *> copies;
  auto it = copies.find(&tw);
  if (it != copies.end()) return it->second;
  int32_t *d = nullptr;
  cudaMalloc(&d, kMaxFFT * sizeof(int32_t));
  cudaMemcpy(d, tw.offset, kMaxFFT * sizeof(int32_t), cudaMemcpyHostToDevice);
  copies[&tw] = d;
  return d;
}

void launch_ragged_tables(const double2 *Trect, int ncanon, int nth, int nphr, const int32_t *rows, const int64_t *off,
                          int64_t K, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  const size_t smem = (size_t)2 * nphr * sizeof(double2);
  cudaFuncSetAttribute(ragged_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  ragged_tables_kernel<<<dim3((unsigned)nth, (unsigned)ncanon), RG_TPB, smem, s>>>(
      Trect, nth, nphr, rows, off, K, tw.d, twiddle_offsets_device(tw), out);
}

void launch_rag2rect(const double2 *in, int64_t in_K, int nth, const int32_t *rows, const int64_t *off, int maxrow,
                     const int32_t *par, const int8_t *oct, const double2 *shift, int64_t nitem, int nphr,
                     double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (nitem <= 0) return;
  const size_t smem = (size_t)2 * maxrow * sizeof(double2);
  cudaFuncSetAttribute(rag2rect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rag2rect_kernel<<<dim3((unsigned)nitem, (unsigned)(nth / 2 + 1)), RG_TPB, smem, s>>>(
      in, in_K, nth, rows, off, par, oct, shift, nphr, tw.d, twiddle_offsets_device(tw), out);
}

void launch_rect2rag(const double2 *in, int nth, int nphr, const int32_t *cbeg, int64_t cbase, const int8_t *oct,
                     const double2 *shift, const double2 *add, const int32_t *rows, const int64_t *off, int64_t K,
                     int64_t nitem, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (nitem <= 0) return;
  const size_t smem = (size_t)3 * nphr * sizeof(double2);
  cudaFuncSetAttribute(rect2rag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rect2rag_kernel<<<dim3((unsigned)nitem, (unsigned)(nth / 2 + 1)), RG_TPB, smem, s>>>(
      in, nth, nphr, cbeg, cbase, oct, shift, add, rows, off, K, tw.d, twiddle_offsets_device(tw), out);
}

}  // namespace hfmm
