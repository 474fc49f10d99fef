// Fourier interpolation / anterpolation on the sphere (product code, sm_100a).
//   P:373-378  interpolation = zero-pad the Fourier coefficients, anterpolation = truncate
//   P:512      kept band |k| <= (min(N, N') - 1) / 2 (Nyquist dropped; R-6)
//   P:724-749  5-step 2-D procedure between quadratures, with eqn:NumSphereSym
//              used to build theta-periodic columns / full phi-rows from half storage.
// Each 1-D resample N -> N' is: forward FFT (length N), spectral pad/truncate with 1/N,
// inverse FFT (length N') computed as the conjugate of a forward FFT of the conjugate (the
// conjugations fold into the pad and the store).
//
// The two-pass layout (rows pass, columns pass, intermediate in global memory / L2):
//   upward   (M2M): rows n <= N_theta/2 resampled N_phi -> N'_phi (step 1), then
//            columns m < N'_phi/2 (step 2) resampled N_theta -> N'_theta (step 3), multiplied by
//            the translation e^{i kappa s.(c_child - c_parent)} and accumulated over the 8
//            children; steps 4-5 are the identity for interpolation (the phi band already fits).
//   downward (L2L): columns of conj(shift) * L_parent (steps 1-2 are the identity for
//            anterpolation) resampled N_theta -> N'_theta (step 3), then rows n <= N'_theta/2
//            rebuilt (step 4) and resampled N_phi -> N'_phi (step 5), + I_child.
//
// Each pass is a tiled, batched FFT kernel: a CTA stages a tile of vectors (RB whole rows, or a
// CB-column strip of one box) in shared memory with coalesced global loads, runs mixed-radix
// Stockham passes (radices 16, 8, 4, 2, 3, 5, 7; radix-16/8 butterflies in registers) with one
// butterfly per thread and the batch index on the fastest thread index -- shared accesses then
// stride over vectors of odd pitch (conflict-free) and the twiddles of a warp are uniform -- and
// writes the tile back with coalesced stores.  Tiles are sized to ~70 KB of shared memory so
// three CTAs share an SM.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "hfmm_impl.h"
#include "fft_regs.cuh"  // c_mul / c_add / ... and the register DFTs dft<R>


namespace hfmm {

void TwiddleSet::build(const std::vector<int> &lengths) {
  for (int i = 0; i < kMaxFFT; ++i) offset[i] = -1;
  std::vector<double2> h;
  for (int N : lengths) {
    if (N <= 0 || N >= kMaxFFT || offset[N] >= 0) continue;
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


// radix codes 0..6 = {16, 8, 4, 2, 3, 5, 7}, 3 bits per pass (a packed word: no local-memory array)
struct RLen {
  int N;
  int nr;
  unsigned codes;
  const double2 *tw;  // e^{-2 pi i t / N}, t < N (global, L1-resident)
};

static RLen rlen(const TwiddleSet &ts, int N, int maxr) {
  RLen L{};
  L.N = N;
  int m = N, e = 0;
  while (m % 2 == 0) m /= 2, ++e;
  auto push = [&](int code) { L.codes |= (unsigned)code << (3 * L.nr++); };
  // powers of two as radix-16 passes plus at most one 8 / 4 (no radix-2 pass unless N has a single 2)
  if (e == 1) push(3);
  else if (maxr < 16) {  // radix-8 passes (fewer registers per thread)
    int e8 = e / 3, rest = e % 3;
    if (rest == 1 && e8 > 0) --e8, push(2), push(2);  // 2^4 = 4 * 4
    for (int i = 0; i < e8; ++i) push(1);
    if (rest == 2) push(2);
  } else {
    int e16 = e / 4, rest = e % 4;
    if (rest == 1 && e16 > 0) --e16, push(1), push(2);  // 2^5 = 8 * 4
    for (int i = 0; i < e16; ++i) push(0);
    if (rest == 2) push(2);
    if (rest == 3) push(1);
  }
  const int odd[3] = {3, 5, 7};
  for (int c = 0; c < 3; ++c)
    while (m % odd[c] == 0) push(4 + c), m /= odd[c];
  L.tw = ts.d + ts.offset[N];
  return L;
}


// ---- integer division by a runtime divisor without the ~25-instruction IDIV sequence: float
//      reciprocal estimate + one correction (exact for 0 <= x < 2^22) -------------------------------
struct FDiv {
  int d;
  float inv;
  __device__ __forceinline__ FDiv(int d_) : d(d_), inv(1.0f / (float)d_) {}
  __device__ __forceinline__ int div(int x, int &rem) const {
    int q = __float2int_rz(__int2float_rz(x) * inv);
    int r = x - q * d;
    if (r < 0) r += d, --q;
    else if (r >= d) r -= d, ++q;
    rem = r;
    return q;
  }
};

// ---- batched vectors: vector v at base v * vstride, element e at base + e * estride ----------------
struct VecSet {
  int nvec, vstride, estride;
};

// Flat index w = o * n + i visited as w = t, t + T, t + 2T, ... (t = threadIdx.x, T = blockDim.x):
// (o, i) advance incrementally -- one division per loop instead of one per element.
struct Walk {
  int o, i, n, dO, dI;
  __device__ __forceinline__ Walk(int t, int T, int n_) : n(n_) {
    o = t / n_, i = t - o * n_;
    dO = T / n_, dI = T - dO * n_;
  }
  __device__ __forceinline__ void next() {
    i += dI, o += dO;
    if (i >= n) i -= n, ++o;
  }
};

template <int R>
__device__ __forceinline__ void stockham_pass(const double2 *__restrict__ src, double2 *__restrict__ dst,
                                              const VecSet &vs, const Walk &w0, int N, int Ns,
                                              const double2 *__restrict__ tw) {
  const int nb = N / R, tstep = N / (Ns * R), es = vs.estride;
  const FDiv fns(Ns);
  // work item w = j * nvec + v: butterfly j of vector v (vector index fastest)
  for (Walk it = w0; it.o < nb; it.next()) {
    const int j = it.o;
    int k;
    fns.div(j, k);
    const int b = it.i * vs.vstride;
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = src[b + (j + r * nb) * es];
    if (Ns > 1) {
      const int kt = k * tstep;
#pragma unroll
      for (int r = 1; r < R; ++r) x[r] = c_mul(x[r], __ldg(&tw[r * kt]));
    }
    dft<R>(x);
    const int o = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[b + (o + r * Ns) * es] = x[r];
  }
}

// forward FFT of every vector (length L.N) in buffer a, ping-pong with b; returns the result buffer
template <int MAXR>
__device__ __forceinline__ double2 *fft_batch(double2 *a, double2 *b, const VecSet &vs, const RLen &L) {
  const Walk w0(threadIdx.x, blockDim.x, vs.nvec);  // (butterfly, vector) walk shared by every pass
  double2 *src = a, *dst = b;
  int Ns = 1;
  for (int s = 0; s < L.nr; ++s) {
    int R;
    switch ((L.codes >> (3 * s)) & 7u) {
      case 0:
        if (MAXR >= 16) stockham_pass<MAXR >= 16 ? 16 : 8>(src, dst, vs, w0, L.N, Ns, L.tw);
        R = 16;
        break;
      case 1: stockham_pass<8>(src, dst, vs, w0, L.N, Ns, L.tw); R = 8; break;
      case 2: stockham_pass<4>(src, dst, vs, w0, L.N, Ns, L.tw); R = 4; break;
      case 3: stockham_pass<2>(src, dst, vs, w0, L.N, Ns, L.tw); R = 2; break;
      case 4: stockham_pass<3>(src, dst, vs, w0, L.N, Ns, L.tw); R = 3; break;
      case 5: stockham_pass<5>(src, dst, vs, w0, L.N, Ns, L.tw); R = 5; break;
      default: stockham_pass<7>(src, dst, vs, w0, L.N, Ns, L.tw); R = 7; break;
    }
    __syncthreads();
    double2 *t = src;
    src = dst;
    dst = t;
    Ns *= R;
  }
  return src;
}

// First pass (Ns = 1) of the inverse transform reading the padded spectrum on the fly: input
// element i < N2 of a vector is conj(X[f] / N) for f = i (i <= N2/2) or i - N2, |f| <= K, else 0
// (R-6) -- the pad never touches shared memory.
template <int R>
__device__ __forceinline__ void stockham_pass_padin(const double2 *__restrict__ X, double2 *__restrict__ dst,
                                                    const VecSet &vs, const Walk &w0, int N, int N2) {
  const int nb = N2 / R, es = vs.estride;
  const int K = (min(N, N2) - 1) / 2;
  const double sc = 1.0 / (double)N;
  for (Walk it = w0; it.o < nb; it.next()) {
    const int j = it.o;
    const int b = it.i * vs.vstride;
    double2 x[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = j + r * nb;
      const int f = (i <= N2 / 2) ? i : i - N2;
      double2 val = make_double2(0.0, 0.0);
      if (f <= K && f >= -K) {
        const double2 y = X[b + (f >= 0 ? f : f + N) * es];
        val = make_double2(y.x * sc, -y.y * sc);
      }
      x[r] = val;
    }
    dft<R>(x);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[b + (j * R + r) * es] = x[r];
  }
}

// inverse resample half: forward FFT (length L.N = N2) of the padded conj spectrum of X (length
// N, in buffer a or b); returns the buffer with the result (conj of the resampled values)
template <int MAXR>
__device__ __forceinline__ double2 *fft_batch_padin(double2 *X, double2 *a, double2 *b, const VecSet &vs,
                                                    const RLen &L, int N) {
  double2 *dst = (X == a) ? b : a;
  const Walk w0(threadIdx.x, blockDim.x, vs.nvec);
  int R0;
  switch (L.codes & 7u) {
    case 0:
      if (MAXR >= 16) stockham_pass_padin<MAXR >= 16 ? 16 : 8>(X, dst, vs, w0, N, L.N);
      R0 = 16;
      break;
    case 1: stockham_pass_padin<8>(X, dst, vs, w0, N, L.N); R0 = 8; break;
    case 2: stockham_pass_padin<4>(X, dst, vs, w0, N, L.N); R0 = 4; break;
    case 3: stockham_pass_padin<2>(X, dst, vs, w0, N, L.N); R0 = 2; break;
    case 4: stockham_pass_padin<3>(X, dst, vs, w0, N, L.N); R0 = 3; break;
    case 5: stockham_pass_padin<5>(X, dst, vs, w0, N, L.N); R0 = 5; break;
    default: stockham_pass_padin<7>(X, dst, vs, w0, N, L.N); R0 = 7; break;
  }
  __syncthreads();
  double2 *src = dst, *nxt = X;
  int Ns = R0;
  for (int s = 1; s < L.nr; ++s) {
    int R;
    switch ((L.codes >> (3 * s)) & 7u) {
      case 0:
        if (MAXR >= 16) stockham_pass<MAXR >= 16 ? 16 : 8>(src, nxt, vs, w0, L.N, Ns, L.tw);
        R = 16;
        break;
      case 1: stockham_pass<8>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 8; break;
      case 2: stockham_pass<4>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 4; break;
      case 3: stockham_pass<2>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 2; break;
      case 4: stockham_pass<3>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 3; break;
      case 5: stockham_pass<5>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 5; break;
      default: stockham_pass<7>(src, nxt, vs, w0, L.N, Ns, L.tw); R = 7; break;
    }
    __syncthreads();
    double2 *t = src;
    src = nxt;
    nxt = t;
    Ns *= R;
  }
  return src;
}

#ifndef HFMM_RS_TPB
#define HFMM_RS_TPB 128
#endif
constexpr int RS_TPB = HFMM_RS_TPB;
#ifndef HFMM_RS_COLS_TPB
#define HFMM_RS_COLS_TPB 128
#endif
#ifndef HFMM_RS_COLS_KB
#define HFMM_RS_COLS_KB 0  // 0: the size plan's budget
#endif
constexpr int RS_COLS_TPB = HFMM_RS_COLS_TPB;

// 16-byte global -> shared copies issued asynchronously (cp.async, L2 only): a thread's whole
// share of a tile is in flight at once instead of one load-store round trip at a time.
__device__ __forceinline__ void cp_async16(double2 *smem, const double2 *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
// ---- rows pass --------------------------------------------------------------------------------
// Row r = (box b, n) for n < nrow = nth/2 + 1 (grid rows n <= N_theta/2).  Input: half storage
// [nth][h] of box b; full row e < nph = (row n)[e] for e < h, (row (nth - n) % nth)[e - h] beyond
// (eqn:NumSphereSym).  UP: output full rows of length nph2 to out[b][n][.]; DOWN: output back to
// half storage out[b][n][t < h2] and out[b][nth - n][t - h2] (+ add).
template <bool UP, int MAXR>
__global__ void __launch_bounds__(RS_TPB) rows_kernel(const double2 *__restrict__ in, int64_t nbox, int nth,
                                                      int nph, int nph2, int RB, int pitch, RLen L1, RLen L2,
                                                      const double2 *__restrict__ add, double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  double2 *A = sm, *Bf = sm + (size_t)RB * pitch;
  const int nrow = nth / 2 + 1, h = nph / 2, h2 = nph2 / 2;
  const int64_t total = nbox * nrow;
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const int nr = (int)min((int64_t)RB, total - r0);
  // load (e fastest: coalesced half-rows); row r0 + v = (box b, grid row n) advanced incrementally
  {
    Walk it(threadIdx.x, blockDim.x, nph);
    int64_t b = (r0 + it.o) / nrow;
    int n = (int)(r0 + it.o - b * nrow);
    while (it.o < nr) {
      const int v = it.o, e = it.i;
      const int row = (e < h || n == 0) ? n : nth - n;
      cp_async16(&A[v * pitch + e], &in[(b * nth + row) * h + (e < h ? e : e - h)]);
      it.next();
      for (n += it.o - v; n >= nrow; n -= nrow) ++b;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const VecSet vs{nr, pitch, 1};
  double2 *X = fft_batch<MAXR>(A, Bf, vs, L1);
  double2 *Z = fft_batch_padin<MAXR>(X, A, Bf, vs, L2, nph);  // conj of the resampled rows
  if (UP) {  // output row r0 + v = (box b, grid row n) is row b * nrow + n of out
    double2 *ob = out + r0 * nph2;
    for (Walk it(threadIdx.x, blockDim.x, nph2); it.o < nr; it.next())
      ob[it.o * nph2 + it.i] = c_conj(Z[it.o * pitch + it.i]);
    return;
  }
  Walk it(threadIdx.x, blockDim.x, nph2);
  int64_t b = (r0 + it.o) / nrow;
  int n = (int)(r0 + it.o - b * nrow);
  for (; it.o < nr;) {
    const int v = it.o, t = it.i;
    double2 val = c_conj(Z[v * pitch + t]);
    {
      int orow = n, oc = t;
      bool st = true;
      if (t >= h2) {
        st = !(n == 0 || 2 * n == nth);   // both halves are the same points
        orow = nth - n, oc = t - h2;
      }
      if (st) {
        const int64_t o = (b * nth + orow) * h2 + oc;
        if (add) val = c_add(val, add[o]);
        out[o] = val;
      }
    }
    it.next();
    for (n += it.o - v; n >= nrow; n -= nrow) ++b;
  }
}

// ---- columns pass -----------------------------------------------------------------------------
// CTA = (item, strip of CB columns).  UP (M2M): item = parent p, columns m < h2 of the rows-pass
// output of each child c in [cbeg[p], cbeg[p+1]) (full rows of length nph2, rows n <= nth/2; the
// theta-periodic column is (row n)[m] for n <= nth/2 and (row nth - n)[m + h2] beyond), resampled
// nth -> nth2, times shift[oct[c]][t][m], summed over the children into out[p][t][m].
// DOWN (L2L): item = child c, columns m < h of conj(shift[oct[c]]) * in[par[c]] ([nth][h]),
// resampled nth -> nth2 into out[c][t][m] ([nth2][h]).
template <bool UP, int MAXR>
__global__ void __launch_bounds__(RS_COLS_TPB) cols_kernel(const double2 *__restrict__ in, int64_t nitem, int nth,
                                                      int ncols, int rowlen, int nth2, int CB, int cp,
                                                      const int32_t *__restrict__ cbeg, int64_t cbase,
                                                      const int32_t *__restrict__ par,
                                                      const int8_t *__restrict__ oct,
                                                      const double2 *__restrict__ shift, RLen L1, RLen L2,
                                                      double2 *__restrict__ out) {
  extern __shared__ double2 sm[];
  const int maxn = max(nth, nth2);
  double2 *A = sm, *Bf = sm + (size_t)maxn * cp;
  const int nstrip = (ncols + CB - 1) / CB;
  const unsigned bq = blockIdx.x / (unsigned)nstrip;  // 32-bit division (grid < 2^32)
  const int64_t item = bq;
  const int m0 = (int)(blockIdx.x - bq * (unsigned)nstrip) * CB;
  const int nc = min(CB, ncols - m0);
  const int64_t c0 = UP ? (cbeg ? cbeg[item] : item) : item;
  const int64_t c1 = UP ? (cbeg ? cbeg[item + 1] : item + 1) : item + 1;
  const VecSet vs{nc, 1, cp};
  for (int64_t c = c0; c < c1; ++c) {
    if (c > c0) __syncthreads();  // previous child's tile consumed
    const int octc = oct ? oct[c] : 0;
    if (UP) {
      const double2 *tb = in + (c - cbase) * (int64_t)(nth / 2 + 1) * rowlen + m0;
      for (Walk it(threadIdx.x, blockDim.x, nc); it.o < nth; it.next()) {
        const int n = it.o, mm = it.i;
        cp_async16(&A[n * cp + mm], (2 * n <= nth) ? &tb[(int64_t)n * rowlen + mm]
                                                   : &tb[(int64_t)(nth - n) * rowlen + mm + ncols]);
      }
    } else {
      const double2 *pb = in + (int64_t)(par ? par[c] : c) * nth * ncols + m0;
      for (Walk it(threadIdx.x, blockDim.x, nc); it.o < nth; it.next())
        cp_async16(&A[it.o * cp + it.i], &pb[(int64_t)it.o * ncols + it.i]);
    }
    cp_async_wait_all();
    __syncthreads();
    if (!UP && shift) {  // e^{i kappa s.(c_parent - c_child)} on the parent grid
      const double2 *sb = shift + (int64_t)octc * nth * ncols + m0;
      for (Walk it(threadIdx.x, blockDim.x, nc); it.o < nth; it.next()) {
        double2 &a = A[it.o * cp + it.i];
        a = c_mul(a, c_conj(__ldg(&sb[it.o * ncols + it.i])));
      }
      __syncthreads();
    }
    double2 *X = fft_batch<MAXR>(A, Bf, vs, L1);
    double2 *Z = fft_batch_padin<MAXR>(X, A, Bf, vs, L2, nth);
    if (UP) {
      double2 *ob = out + item * nth2 * (int64_t)ncols + m0;
      const double2 *sb = shift ? shift + (int64_t)octc * nth2 * ncols + m0 : nullptr;
      for (Walk it(threadIdx.x, blockDim.x, nc); it.o < nth2; it.next()) {
        const int t = it.o, mm = it.i;
        double2 v = c_conj(Z[t * cp + mm]);
        if (sb) v = c_mul(v, sb[t * ncols + mm]);
        double2 &o = ob[(int64_t)t * ncols + mm];
        o = (c == c0) ? v : c_add(o, v);   // same thread owns o for every child
      }
    } else {
      double2 *ob = out + c * nth2 * (int64_t)ncols + m0;
      for (Walk it(threadIdx.x, blockDim.x, nc); it.o < nth2; it.next())
        ob[(int64_t)it.o * ncols + it.i] = c_conj(Z[it.o * cp + it.i]);
    }
  }
}

// Resident CTAs per SM asked of ptxas by the register-resident passes (A/B, C2 same box,
// profiles/r02/rs2_minb_ab.txt): the downward passes and the upward rows pass fit 4 CTAs per SM
// in shared memory and gain from the extra warps (B32 anterp 5.22 -> 4.67 ms, L2L 7.19 -> 6.04 ms,
// interp 4.94 -> 4.87 ms); the upward column pass (cp.async staging, 64 KB) stays at 3 per SM,
// where the 128-register cap only adds spills (B64 interp 16.9 -> 17.5 ms, M2M 20.2 -> 21.8 ms).
#ifndef HFMM_RS2_MINB_UP
#define HFMM_RS2_MINB_UP 3
#endif
#ifndef HFMM_RS2_MINB_UPROWS
#define HFMM_RS2_MINB_UPROWS 4
#endif
#ifndef HFMM_RS2_MINB_DN
#define HFMM_RS2_MINB_DN 4
#endif
#ifndef HFMM_RS2_REGACC
#define HFMM_RS2_REGACC 1   // M2M column pass on power-of-two grids: sum the 8 children in registers (ACC
                            // flavour; 2 CTAs/SM at 256 points) instead of through the output (A/B
                            // profiles/r02/regacc_ab.txt: C2 B32 M2M 5.29 -> 5.11 ms, B64 20.1 -> 18.6-19.0 ms)
#endif
// ... for the power-of-two sizes (C2 grids) only: on the 7-smooth grids of the matvec configs the
// extra CTAs per SM cost C3 0.45 ms per matvec next to the concurrent near field (3.74 -> 4.2 ms,
// same box, profiles/r02/l2t_ab.txt "oldlb"), so those instantiations keep 3.
constexpr bool rs2_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
template <bool UP, bool ROWS, int N, int N2>
constexpr int rs2_minb() {
  return !(rs2_pow2(N) && rs2_pow2(N2)) ? 3 : UP ? (ROWS ? HFMM_RS2_MINB_UPROWS : HFMM_RS2_MINB_UP) : HFMM_RS2_MINB_DN;
}
// ---- register-resident two-level resample passes ----------------------------------------------
// A 1-D resample N -> N' with N = N1 N2 and N' = M1 M2 (factors: register DFT sizes) by one group of
// G lanes (G = the largest factor) inside a warp, data in registers between the passes:
//   forward N:  lane n2 < N2 holds x[N2 n1 + n2] (n1 < N1): DFT_N1, twiddle w_N^{n2 k1}; exchange;
//               lane k1 < N1 holds the N2 values: DFT_N2 -> X[k1 + N1 k2];
//   pad:        X through the group's shared buffer; lane m2 < M2 reads Z[M2 m1 + m2] =
//               conj(X[f]) / N for the kept band |f| <= K (R-6), else 0;
//   forward N': the same two stages on Z; conj of the result = the resampled vector.
// Three __syncwarp exchanges per vector instead of one shared round trip per radix pass.
template <bool UP, int FN1, int FN2, int IN1, int IN2>
__global__ void __launch_bounds__(128, (rs2_minb<UP, true, FN1 * FN2, IN1 * IN2>())) rows2_kernel(const double2 *__restrict__ in, int64_t nbox, int nth,
                                                      const double2 *__restrict__ twN,
                                                      const double2 *__restrict__ twN2,
                                                      const double2 *__restrict__ add, double2 *__restrict__ out) {
  constexpr int N = FN1 * FN2, N2 = IN1 * IN2;
  constexpr int GM = (FN1 > IN1 ? FN1 : IN1) > (FN2 > IN2 ? FN2 : IN2) ? (FN1 > IN1 ? FN1 : IN1) : (FN2 > IN2 ? FN2 : IN2);
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;  // lanes per group (divides 32)
  constexpr int BF = FN1 * (FN2 + 1), BI = IN1 * (IN2 + 1);
  constexpr int BUFW = (BF > BI ? BF : BI) > (N > N2 ? N : N2) ? (BF > BI ? BF : BI) : (N > N2 ? N : N2);
  constexpr int VW = 32 / G;
  extern __shared__ double2 sm[];
  double2 *tw1 = sm, *tw2 = sm + N;           // w_N^j, w_N'^j
  double2 *bufs = sm + N + N2;
  for (int j = threadIdx.x; j < N; j += blockDim.x) tw1[j] = twN[j];
  for (int j = threadIdx.x; j < N2; j += blockDim.x) tw2[j] = twN2[j];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, g = lane - grp * G;
  double2 *buf = bufs + (size_t)(warp * VW + grp) * BUFW;
  const int nrow = nth / 2 + 1;
  constexpr int h = N / 2;
  const int64_t total = nbox * nrow;
  constexpr int K = ((N < N2 ? N : N2) - 1) / 2;
  constexpr double sc = 1.0 / (double)N;
  const int64_t vstep = (int64_t)gridDim.x * (blockDim.x >> 5) * VW;
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * VW; r0 < total; r0 += vstep) {
    const int64_t r = r0 + grp;
    const bool vok = r < total;
    const int64_t b = vok ? r / nrow : 0;
    const int n = vok ? (int)(r - b * nrow) : 0;
    double2 x[16];
    // forward N, stage 1: lane g < FN2 loads elements e = FN2 n1 + g of the full row (eqn:NumSphereSym)
    if (vok && g < FN2) {
      const double2 *lo = in + (b * nth + n) * h, *hi = in + (b * nth + (n == 0 ? 0 : nth - n)) * h;
#pragma unroll
      for (int n1 = 0; n1 < FN1; ++n1) {
        const int e = FN2 * n1 + g;
        x[n1] = e < h ? lo[e] : hi[e - h];
      }
      dft<FN1>(x);
#pragma unroll
      for (int k1 = 1; k1 < FN1; ++k1) x[k1] = c_mul(x[k1], tw1[g * k1]);
#pragma unroll
      for (int k1 = 0; k1 < FN1; ++k1) buf[k1 * (FN2 + 1) + g] = x[k1];
    }
    __syncwarp();
    if (vok && g < FN1) {  // stage 2: lane k1 -> X[k1 + FN1 k2]
#pragma unroll
      for (int n2 = 0; n2 < FN2; ++n2) x[n2] = buf[g * (FN2 + 1) + n2];
    }
    __syncwarp();
    if (vok && g < FN1) {
      dft<FN2>(x);
#pragma unroll
      for (int k2 = 0; k2 < FN2; ++k2) buf[g + FN1 * k2] = x[k2];
    }
    __syncwarp();
    if (vok && g < IN2) {  // padded conj spectrum: lane g holds Z[IN2 m1 + g]
#pragma unroll
      for (int m1 = 0; m1 < IN1; ++m1) {
        const int i = IN2 * m1 + g;
        const int f = (i <= N2 / 2) ? i : i - N2;
        double2 z = make_double2(0.0, 0.0);
        if (f <= K && f >= -K) {
          const double2 y = buf[f >= 0 ? f : f + N];
          z = make_double2(y.x * sc, -y.y * sc);
        }
        x[m1] = z;
      }
    }
    __syncwarp();
    if (vok && g < IN2) {
      dft<IN1>(x);
#pragma unroll
      for (int k1 = 1; k1 < IN1; ++k1) x[k1] = c_mul(x[k1], tw2[g * k1]);
#pragma unroll
      for (int k1 = 0; k1 < IN1; ++k1) buf[k1 * (IN2 + 1) + g] = x[k1];
    }
    __syncwarp();
    if (vok && g < IN1) {
#pragma unroll
      for (int n2 = 0; n2 < IN2; ++n2) x[n2] = buf[g * (IN2 + 1) + n2];
      dft<IN2>(x);
      if (UP) {  // full row n of box b
        double2 *o = out + r * N2;
#pragma unroll
        for (int k2 = 0; k2 < IN2; ++k2) o[g + IN1 * k2] = c_conj(x[k2]);
      } else {   // back to half storage: t < N2/2 -> row n, beyond -> row nth - n (+ add)
        constexpr int h2 = N2 / 2;
        const bool mirror = !(n == 0 || 2 * n == nth);
#pragma unroll
        for (int k2 = 0; k2 < IN2; ++k2) {
          const int t = g + IN1 * k2;
          if (t >= h2 && !mirror) continue;   // both halves are the same points
          const int64_t o = (b * nth + (t < h2 ? n : nth - n)) * h2 + (t < h2 ? t : t - h2);
          double2 val = c_conj(x[k2]);
          if (add) val = c_add(val, add[o]);
          out[o] = val;
        }
      }
    }
    __syncwarp();
  }
}

// Register-resident two-level columns pass.  CTA = 4 warps = CW = 8 columns (lane & 7) x 16 group
// lanes (g = 4 warp + lane / 8): every global access of a warp is 4 runs of 8 consecutive columns.
// UP (M2M / interpolation): unit = (parent, strip); children c in [cbeg[p], cbeg[p+1]) (or the box
// itself) resampled nth -> nth2 along theta, times shift[oct[c]], summed in registers, stored once.
// DOWN (L2L / anterpolation): unit = (child c, strip) of conj(shift[oct[c]]) * in[par[c]].
constexpr int RS2_CW = 8, RS2_CWP = 9;

template <bool UP, int FN1, int FN2, int IN1, int IN2, bool ACC = false>
__global__ void __launch_bounds__(128, (ACC ? (IN1 * IN2 >= 256 ? 2 : 3) : rs2_minb<UP, false, FN1 * FN2, IN1 * IN2>()))
cols2_kernel(const double2 *__restrict__ in, int64_t nitem, int ncols,
                                                   int rowlen, const int32_t *__restrict__ cbeg, int64_t cbase,
                                                   const int32_t *__restrict__ par, const int8_t *__restrict__ oct,
                                                   const double2 *__restrict__ shift,
                                                   const double2 *__restrict__ twN,
                                                   const double2 *__restrict__ twN2, double2 *__restrict__ out) {
  constexpr int N = FN1 * FN2, N2 = IN1 * IN2;
  constexpr int BUFR = Max2<Max2<FN1 * (FN2 + 1), IN1 * (IN2 + 1)>::v, Max2<N, N2>::v>::v;
  extern __shared__ double2 sm[];
  double2 *tw1 = sm, *tw2 = sm + N, *buf = sm + N + N2;
  for (int j = threadIdx.x; j < N; j += blockDim.x) tw1[j] = twN[j];
  for (int j = threadIdx.x; j < N2; j += blockDim.x) tw2[j] = twN2[j];
  const int v = threadIdx.x & (RS2_CW - 1), g = threadIdx.x >> 3;  // column in strip, group lane
  const int nstrip = (ncols + RS2_CW - 1) / RS2_CW;
  constexpr int K = ((N < N2 ? N : N2) - 1) / 2;
  constexpr double sc = 1.0 / (double)N;
  const int64_t nunit = nitem * nstrip;
  // Steps (unit u, child c) in CTA order.  Upward: the input strip of the next step is fetched into
  // `stg` with cp.async while the current one is transformed (hides the global-memory latency;
  // same-box A/B: C2 B64 interp 20.1 -> 17.6 ms).  Downward the extra 37 KB cost a CTA per SM
  // (B64 anterp 16.8 -> 19.0 ms), so it loads straight into registers.
  constexpr bool PF = UP;
  double2 *stg = buf + BUFR * RS2_CWP;  // [N][CWP] (PF only)
  auto crange = [&](int64_t uu, int64_t &a0, int64_t &a1) {
    const int64_t it = uu / nstrip;
    a0 = it, a1 = it + 1;
    if (UP && cbeg) a0 = cbeg[it], a1 = cbeg[it + 1];
  };
  auto issue = [&](int64_t uu, int64_t cc) {
    const int64_t it = uu / nstrip;
    const int mb = (int)(uu - it * nstrip) * RS2_CW;
    const double2 *cb = UP ? in + (cc - cbase) * (int64_t)(N / 2 + 1) * rowlen
                           : in + (int64_t)(par ? par[cc] : cc) * N * ncols;
    for (int e = threadIdx.x; e < N * RS2_CW; e += blockDim.x) {
      const int n = e >> 3, vv = e & (RS2_CW - 1), mm = mb + vv;
      if (mm >= ncols) continue;
      const double2 *src = UP ? ((2 * n <= N) ? &cb[(int64_t)n * rowlen + mm] : &cb[(int64_t)(N - n) * rowlen + mm + ncols])
                              : &cb[(int64_t)n * ncols + mm];
      cp_async16(&stg[n * RS2_CWP + vv], src);
    }
  };
  int64_t u = blockIdx.x;
  if (u >= nunit) return;
  int64_t c0, c1;
  crange(u, c0, c1);
  double2 acc[ACC ? IN2 : 1];   // ACC (M2M): the unit's child sum (this thread's outputs)
  int64_t c = c0;
  if (PF) issue(u, c);
  for (;;) {
    const int64_t item = u / nstrip;
    const int m = (int)(u - item * nstrip) * RS2_CW + v;
    const bool mok = m < ncols;
    int64_t nu = u, nc = c + 1, n0 = c0, n1_ = c1;  // next step
    {
      double2 x[16];
      if (PF) cp_async_wait_all();
      __syncthreads();  // stg holds step (u, c); previous use of buf done; twiddles staged
      if (g < FN2) {     // forward nth, stage 1: x[n1] = column element FN2 n1 + g
        if (PF) {
#pragma unroll
          for (int n1 = 0; n1 < FN1; ++n1) x[n1] = mok ? stg[(FN2 * n1 + g) * RS2_CWP + v] : make_double2(0.0, 0.0);
        } else {  // all loads of the column first (no branch between them: one latency per column)
          const double2 *cb = UP ? in + (c - cbase) * (int64_t)(N / 2 + 1) * rowlen
                                 : in + (int64_t)(par ? par[c] : c) * N * ncols;
#pragma unroll
          for (int n1 = 0; n1 < FN1; ++n1) {
            const int n = FN2 * n1 + g;
            const int64_t o = UP ? ((2 * n <= N) ? (int64_t)n * rowlen + m : (int64_t)(N - n) * rowlen + m + ncols)
                                 : (int64_t)n * ncols + m;
            x[n1] = mok ? cb[o] : make_double2(0.0, 0.0);
          }
        }
        if (!UP && shift && mok) {
          const double2 *sb = shift + (int64_t)(oct ? oct[c] : 0) * N * ncols;
          double2 t[FN1];
#pragma unroll
          for (int n1 = 0; n1 < FN1; ++n1) t[n1] = __ldg(&sb[(int64_t)(FN2 * n1 + g) * ncols + m]);
#pragma unroll
          for (int n1 = 0; n1 < FN1; ++n1) x[n1] = c_mul(x[n1], c_conj(t[n1]));
        }
        dft<FN1>(x);
#pragma unroll
        for (int k1 = 1; k1 < FN1; ++k1) x[k1] = c_mul(x[k1], tw1[g * k1]);
#pragma unroll
        for (int k1 = 0; k1 < FN1; ++k1) buf[(k1 * (FN2 + 1) + g) * RS2_CWP + v] = x[k1];
      }
      __syncthreads();  // stg consumed: fetch the next step's strip
      if (nc >= c1) {
        nu = u + gridDim.x;
        if (nu < nunit) crange(nu, n0, n1_), nc = n0;
      }
      if (PF && nu < nunit) issue(nu, nc);
      if (g < FN1) {
#pragma unroll
        for (int n2 = 0; n2 < FN2; ++n2) x[n2] = buf[(g * (FN2 + 1) + n2) * RS2_CWP + v];
      }
      __syncthreads();
      if (g < FN1) {
        dft<FN2>(x);
#pragma unroll
        for (int k2 = 0; k2 < FN2; ++k2) buf[(g + FN1 * k2) * RS2_CWP + v] = x[k2];
      }
      __syncthreads();
      if (g < IN2) {  // padded / truncated conj spectrum: Z[IN2 m1 + g]
#pragma unroll
        for (int m1 = 0; m1 < IN1; ++m1) {
          const int i = IN2 * m1 + g;
          const int f = (i <= N2 / 2) ? i : i - N2;
          double2 z = make_double2(0.0, 0.0);
          if (f <= K && f >= -K) {
            const double2 y = buf[(f >= 0 ? f : f + N) * RS2_CWP + v];
            z = make_double2(y.x * sc, -y.y * sc);
          }
          x[m1] = z;
        }
      }
      __syncthreads();
      if (g < IN2) {
        dft<IN1>(x);
#pragma unroll
        for (int k1 = 1; k1 < IN1; ++k1) x[k1] = c_mul(x[k1], tw2[g * k1]);
#pragma unroll
        for (int k1 = 0; k1 < IN1; ++k1) buf[(k1 * (IN2 + 1) + g) * RS2_CWP + v] = x[k1];
      }
      __syncthreads();
      if (g < IN1) {
#pragma unroll
        for (int n2 = 0; n2 < IN2; ++n2) x[n2] = buf[(g * (IN2 + 1) + n2) * RS2_CWP + v];
        dft<IN2>(x);
        if (UP) {
          if (mok) {  // shift and sum over the children (same thread owns the outputs for every child)
            double2 *ob = out + item * (int64_t)N2 * ncols + m;
#pragma unroll
            for (int k2 = 0; k2 < IN2; ++k2) x[k2] = c_conj(x[k2]);
            if (shift) {
              const double2 *sb = shift + (int64_t)(oct ? oct[c] : 0) * N2 * ncols + m;
              double2 t[IN2];
#pragma unroll
              for (int k2 = 0; k2 < IN2; ++k2) t[k2] = __ldg(&sb[(int64_t)(g + IN1 * k2) * ncols]);
#pragma unroll
              for (int k2 = 0; k2 < IN2; ++k2) x[k2] = c_mul(x[k2], t[k2]);
            }
            if constexpr (ACC) {
            // children summed in registers; one store after the unit's last child
#pragma unroll
            for (int k2 = 0; k2 < IN2; ++k2) acc[k2] = (c != c0) ? c_add(acc[k2], x[k2]) : x[k2];
            if (c + 1 == c1) {
#pragma unroll
              for (int k2 = 0; k2 < IN2; ++k2) ob[(int64_t)(g + IN1 * k2) * ncols] = acc[k2];
            }
            } else {
            if (c != c0) {
              double2 t[IN2];
#pragma unroll
              for (int k2 = 0; k2 < IN2; ++k2) t[k2] = ob[(int64_t)(g + IN1 * k2) * ncols];
#pragma unroll
              for (int k2 = 0; k2 < IN2; ++k2) x[k2] = c_add(x[k2], t[k2]);
            }
#pragma unroll
            for (int k2 = 0; k2 < IN2; ++k2) ob[(int64_t)(g + IN1 * k2) * ncols] = x[k2];
            }
          }
        } else if (mok) {
          double2 *ob = out + c * (int64_t)N2 * ncols + m;
#pragma unroll
          for (int k2 = 0; k2 < IN2; ++k2) ob[(int64_t)(g + IN1 * k2) * ncols] = c_conj(x[k2]);
        }
      }
    }
    if (nu >= nunit) break;
    u = nu, c = nc, c0 = n0, c1 = n1_;
  }
}

template <bool UP, int FN1, int FN2, int IN1, int IN2>
static void launch_cols2_t(const double2 *in, int64_t nitem, int ncols, int rowlen, const int32_t *cbeg,
                           int64_t cbase, const int32_t *par, const int8_t *oct, const double2 *shift, double2 *out,
                           const TwiddleSet &tw, cudaStream_t s) {
  constexpr int N = FN1 * FN2, N2 = IN1 * IN2;
  constexpr int BUFR = Max2<Max2<FN1 * (FN2 + 1), IN1 * (IN2 + 1)>::v, Max2<N, N2>::v>::v;
  const size_t smem = ((size_t)N + N2 + (size_t)(BUFR + (UP ? N : 0)) * RS2_CWP) * sizeof(double2);
  auto kern = cols2_kernel<UP, FN1, FN2, IN1, IN2, false>;
  if constexpr (UP && rs2_pow2(FN1 * FN2) && rs2_pow2(IN1 * IN2))
    if (HFMM_RS2_REGACC && cbeg) kern = cols2_kernel<UP, FN1, FN2, IN1, IN2, true>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
  const int64_t nunit = nitem * ((ncols + RS2_CW - 1) / RS2_CW);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nunit, (int64_t)nsm * std::max(per, 1)));
  kern<<<grid, 128, smem, s>>>(in, nitem, ncols, rowlen, cbeg, cbase, par, oct, shift, tw.d + tw.offset[N],
                               tw.d + tw.offset[N2], out);
}

static int rs2_enabled() {
  static const int enabled = [] {   // thread-safe one-time initialisation
    const char *e = getenv("HFMM_RS2");   // 0: tiled passes only (A/B)
    return e ? atoi(e) : 1;
  }();
  return enabled;
}

// (nth, nth2) pairs with a register-resident columns pass; false: use the tiled kernel
template <bool UP>
static bool launch_cols2(const double2 *in, int64_t nitem, int nth, int ncols, int rowlen, int nth2,
                         const int32_t *cbeg, int64_t cbase, const int32_t *par, const int8_t *oct,
                         const double2 *shift, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  // size floor (same-box A/Bs on the power-of-two C2 grids); the 7-smooth matvec pairs always take the
  // register-resident pass when instantiated (C3 / C5 54 -> 120 upward: the tiled column pass took 3x
  // the time of the downward cols2 pass, profiles/r02/launches_c3_r02f.csv)
  if (!rs2_enabled() || (std::max(nth, nth2) < (UP ? 128 : 64) && rs2_pow2(nth) && rs2_pow2(nth2))) return false;
  switch (nth * 1000 + nth2) {
#define RS2C(a, b, F1, F2, I1, I2) \
  case a * 1000 + b: launch_cols2_t<UP, F1, F2, I1, I2>(in, nitem, ncols, rowlen, cbeg, cbase, par, oct, shift, out, tw, s); return true;
    RS2C(16, 32, 4, 4, 8, 4)
    RS2C(32, 64, 8, 4, 8, 8)
    RS2C(64, 128, 8, 8, 16, 8)
    RS2C(128, 256, 16, 8, 16, 16)
    RS2C(32, 16, 8, 4, 4, 4)
    RS2C(64, 32, 8, 8, 8, 4)
    RS2C(128, 64, 16, 8, 8, 8)
    RS2C(256, 128, 16, 16, 16, 8)
    // 7-smooth grids of the BASELINE matvec configs (C3: 54 <-> 120, C4: 60 <-> 140 <-> 240,
    // C5: 54 <-> 120; factors from the register DFTs incl. the composite 6, 9, 10, 12, 14, 15)
    RS2C(54, 120, 9, 6, 12, 10)
    RS2C(120, 54, 12, 10, 9, 6)
    RS2C(60, 140, 10, 6, 14, 10)
    RS2C(140, 60, 14, 10, 10, 6)
    RS2C(140, 240, 14, 10, 16, 15)
    RS2C(240, 140, 16, 15, 14, 10)
    // accuracy-policy plans (tau = eps/10; C3_acc / C5_acc: 90x96 <-> 150x160)
    RS2C(90, 150, 10, 9, 15, 10)
    RS2C(150, 90, 15, 10, 10, 9)
    RS2C(40, 90, 8, 5, 10, 9)     // two-pass alternative to box2 40 <-> 90x96 (HFMM_BOX2_4090=0)
    RS2C(90, 40, 10, 9, 8, 5)
#undef RS2C
    default: return false;
  }
}

template <bool UP, int FN1, int FN2, int IN1, int IN2>
static void launch_rows2_t(const double2 *in, int64_t nbox, int nth, const double2 *add, double2 *out,
                           const TwiddleSet &tw, cudaStream_t s) {
  constexpr int N = FN1 * FN2, N2 = IN1 * IN2;
  constexpr int GM = std::max(std::max(FN1, FN2), std::max(IN1, IN2));
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  constexpr int BUFW = std::max(std::max(FN1 * (FN2 + 1), IN1 * (IN2 + 1)), std::max(N, N2));
  constexpr int VW = 32 / G, warps = 4;
  const size_t smem = ((size_t)N + N2 + (size_t)warps * VW * BUFW) * sizeof(double2);
  auto kern = rows2_kernel<UP, FN1, FN2, IN1, IN2>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 32 * warps, smem);
  const int64_t total = nbox * (nth / 2 + 1);
  const int64_t need = (total + (int64_t)warps * VW - 1) / ((int64_t)warps * VW);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * std::max(per, 1)));
  kern<<<grid, 32 * warps, smem, s>>>(in, nbox, nth, tw.d + tw.offset[N], tw.d + tw.offset[N2], add, out);
}

// Per-size plan of the register-resident passes (same-box A/Bs, profiles/r01/rs2_ab*.txt): rows
// passes and downward column passes from 64-point grids up, upward column passes from 128.
template <bool UP>
static bool launch_rows2(const double2 *in, int64_t nbox, int nth, int nph, int nph2, const double2 *add,
                         double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (!rs2_enabled() || std::max(nph, nph2) < 64) return false;
  switch (nph * 1000 + nph2) {
#define RS2R(a, b, F1, F2, I1, I2) \
  case a * 1000 + b: launch_rows2_t<UP, F1, F2, I1, I2>(in, nbox, nth, add, out, tw, s); return true;
    RS2R(32, 64, 8, 4, 8, 8)
    RS2R(64, 128, 8, 8, 16, 8)
    RS2R(128, 256, 16, 8, 16, 16)
    RS2R(64, 32, 8, 8, 8, 4)
    RS2R(128, 64, 16, 8, 8, 8)
    RS2R(256, 128, 16, 16, 16, 8)
    RS2R(56, 120, 8, 7, 12, 10)
    RS2R(120, 56, 12, 10, 8, 7)
    RS2R(60, 140, 10, 6, 14, 10)
    RS2R(140, 60, 14, 10, 10, 6)
    RS2R(140, 240, 14, 10, 16, 15)
    RS2R(240, 140, 16, 15, 14, 10)
    RS2R(96, 160, 12, 8, 16, 10)
    RS2R(160, 96, 16, 10, 12, 8)
    RS2R(40, 96, 8, 5, 12, 8)
    RS2R(96, 40, 12, 8, 8, 5)
#undef RS2R
    default: return false;
  }
}

// ---- single-pass upward resample for small grids (interpolation / M2M) --------------------------
// One CTA per item (a box, or a parent with its children): for each child the row pass (register
// two-level transforms, a lane group per row) writes the resampled full rows into a shared-memory
// intermediate, then the column pass (8 columns x 16 group lanes per 4 warps) reads the theta-
// periodic columns from it and stores the shifted (and child-summed) parent field.  The
// intermediate never leaves the SM: HBM traffic is the algorithmic read-child + write-parent.
// Column strips of the single-pass kernels: CW columns x GC group lanes per 128 threads, GC the
// power of two covering the column DFT factors -- 8 lanes (16 columns) when every factor is <= 8,
// so the stages with 4-6 active lanes no longer idle half of a 16-lane group (HFMM_BOX2_WIDE=0: the
// previous 8 x 16 strips).
#ifndef HFMM_BOX2_WIDE
#define HFMM_BOX2_WIDE 1
#endif
template <int CF1, int CF2, int CI1, int CI2>
struct Box2Cols {
  static constexpr int GM = Max2<Max2<CF1, CF2>::v, Max2<CI1, CI2>::v>::v;
  static constexpr int GC = (HFMM_BOX2_WIDE && GM <= 8) ? 8 : 16;
  static constexpr int CW = 128 / GC, CWP = CW + 1;
};

template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
__global__ void __launch_bounds__(128) box2_up_kernel(const double2 *__restrict__ in, int64_t nitem,
                                                     const int32_t *__restrict__ cbeg, int64_t cbase,
                                                     const int8_t *__restrict__ oct,
                                                     const double2 *__restrict__ shift,
                                                     const double2 *__restrict__ twR, const double2 *__restrict__ twR2,
                                                     const double2 *__restrict__ twC, const double2 *__restrict__ twC2,
                                                     double2 *__restrict__ out) {
  constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2;   // nph -> nph2 (rows)
  constexpr int NC = CF1 * CF2, NC2 = CI1 * CI2;   // nth -> nth2 (columns)
  using BC = Box2Cols<CF1, CF2, CI1, CI2>;
  constexpr int h = NR / 2, h2 = NR2 / 2, nrow = NC / 2 + 1;
  constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  constexpr int VW = 32 / G;
  constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  constexpr int IP = NR2 + 1;                      // intermediate row pitch
  constexpr int KR = ((NR < NR2 ? NR : NR2) - 1) / 2, KC = ((NC < NC2 ? NC : NC2) - 1) / 2;
  extern __shared__ double2 sm[];
  double2 *tr1 = sm, *tr2 = tr1 + NR, *tc1 = tr2 + NR2, *tc2 = tc1 + NC;
  double2 *inter = tc2 + NC2;                      // [nrow][IP]
  double2 *rbuf = inter + nrow * IP;               // [4 warps][VW][RBUF]
  double2 *cbuf = rbuf + 4 * VW * RBUF;            // [CBUF][BC::CWP]
  for (int j = threadIdx.x; j < NR; j += blockDim.x) tr1[j] = twR[j];
  for (int j = threadIdx.x; j < NR2; j += blockDim.x) tr2[j] = twR2[j];
  for (int j = threadIdx.x; j < NC; j += blockDim.x) tc1[j] = twC[j];
  for (int j = threadIdx.x; j < NC2; j += blockDim.x) tc2[j] = twC2[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, gr = lane - grp * G;   // row pass: lane group, lane in group
  double2 *rb = rbuf + (warp * VW + grp) * RBUF;
  const int v = threadIdx.x % BC::CW, g = threadIdx.x / BC::CW;  // column pass
  for (int64_t item = blockIdx.x; item < nitem; item += gridDim.x) {
    int64_t c0 = item, c1 = item + 1;
    if (cbeg) c0 = cbeg[item], c1 = cbeg[item + 1];
    for (int64_t c = c0; c < c1; ++c) {
      double2 x[16];
      __syncthreads();  // twiddles staged / previous child's intermediate consumed
      // ---- rows n <= nth/2 of child c: nph -> nph2, into inter[n][.] ----
      for (int r0 = warp * VW; r0 < nrow; r0 += 4 * VW) {
        const int n = r0 + grp;
        const bool vok = n < nrow && grp < VW;
        if (vok && gr < RF2) {
          const double2 *lo = in + ((c - cbase) * NC + n) * h, *hi = in + ((c - cbase) * NC + (n == 0 ? 0 : NC - n)) * h;
#pragma unroll
          for (int n1 = 0; n1 < RF1; ++n1) {
            const int e = RF2 * n1 + gr;
            x[n1] = e < h ? lo[e] : hi[e - h];
          }
          dft<RF1>(x);
#pragma unroll
          for (int k1 = 1; k1 < RF1; ++k1) x[k1] = c_mul(x[k1], tr1[gr * k1]);
#pragma unroll
          for (int k1 = 0; k1 < RF1; ++k1) rb[k1 * (RF2 + 1) + gr] = x[k1];
        }
        __syncwarp();
        if (vok && gr < RF1) {
#pragma unroll
          for (int n2 = 0; n2 < RF2; ++n2) x[n2] = rb[gr * (RF2 + 1) + n2];
        }
        __syncwarp();
        if (vok && gr < RF1) {
          dft<RF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < RF2; ++k2) rb[gr + RF1 * k2] = x[k2];
        }
        __syncwarp();
        if (vok && gr < RI2) {
#pragma unroll
          for (int m1 = 0; m1 < RI1; ++m1) {
            const int i = RI2 * m1 + gr;
            const int f = (i <= NR2 / 2) ? i : i - NR2;
            double2 z = make_double2(0.0, 0.0);
            if (f <= KR && f >= -KR) {
              const double2 y = rb[f >= 0 ? f : f + NR];
              z = make_double2(y.x * (1.0 / NR), -y.y * (1.0 / NR));
            }
            x[m1] = z;
          }
        }
        __syncwarp();
        if (vok && gr < RI2) {
          dft<RI1>(x);
#pragma unroll
          for (int k1 = 1; k1 < RI1; ++k1) x[k1] = c_mul(x[k1], tr2[gr * k1]);
#pragma unroll
          for (int k1 = 0; k1 < RI1; ++k1) rb[k1 * (RI2 + 1) + gr] = x[k1];
        }
        __syncwarp();
        if (vok && gr < RI1) {
#pragma unroll
          for (int n2 = 0; n2 < RI2; ++n2) x[n2] = rb[gr * (RI2 + 1) + n2];
          dft<RI2>(x);
#pragma unroll
          for (int k2 = 0; k2 < RI2; ++k2) inter[n * IP + gr + RI1 * k2] = c_conj(x[k2]);
        }
        __syncwarp();
      }
      // ---- columns m < h2 of the intermediate: nth -> nth2, shift, sum into the parent ----
      for (int m0 = 0; m0 < h2; m0 += BC::CW) {
        const int m = m0 + v;
        const bool mok = m < h2;
        __syncthreads();  // intermediate complete / previous strip's cbuf consumed
        if (g < CF2) {
#pragma unroll
          for (int n1 = 0; n1 < CF1; ++n1) {
            const int nn = CF2 * n1 + g;
            x[n1] = mok ? ((2 * nn <= NC) ? inter[nn * IP + m] : inter[(NC - nn) * IP + m + h2])
                        : make_double2(0.0, 0.0);
          }
          dft<CF1>(x);
#pragma unroll
          for (int k1 = 1; k1 < CF1; ++k1) x[k1] = c_mul(x[k1], tc1[g * k1]);
#pragma unroll
          for (int k1 = 0; k1 < CF1; ++k1) cbuf[(k1 * (CF2 + 1) + g) * BC::CWP + v] = x[k1];
        }
        __syncthreads();
        if (g < CF1) {
#pragma unroll
          for (int n2 = 0; n2 < CF2; ++n2) x[n2] = cbuf[(g * (CF2 + 1) + n2) * BC::CWP + v];
        }
        __syncthreads();
        if (g < CF1) {
          dft<CF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < CF2; ++k2) cbuf[(g + CF1 * k2) * BC::CWP + v] = x[k2];
        }
        __syncthreads();
        if (g < CI2) {
#pragma unroll
          for (int m1 = 0; m1 < CI1; ++m1) {
            const int i = CI2 * m1 + g;
            const int f = (i <= NC2 / 2) ? i : i - NC2;
            double2 z = make_double2(0.0, 0.0);
            if (f <= KC && f >= -KC) {
              const double2 y = cbuf[(f >= 0 ? f : f + NC) * BC::CWP + v];
              z = make_double2(y.x * (1.0 / NC), -y.y * (1.0 / NC));
            }
            x[m1] = z;
          }
        }
        __syncthreads();
        if (g < CI2) {
          dft<CI1>(x);
#pragma unroll
          for (int k1 = 1; k1 < CI1; ++k1) x[k1] = c_mul(x[k1], tc2[g * k1]);
#pragma unroll
          for (int k1 = 0; k1 < CI1; ++k1) cbuf[(k1 * (CI2 + 1) + g) * BC::CWP + v] = x[k1];
        }
        __syncthreads();
        if (g < CI1 && mok) {
#pragma unroll
          for (int n2 = 0; n2 < CI2; ++n2) x[n2] = cbuf[(g * (CI2 + 1) + n2) * BC::CWP + v];
          dft<CI2>(x);
          double2 *ob = out + item * (int64_t)NC2 * h2 + m;
#pragma unroll
          for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_conj(x[k2]);
          if (shift) {
            const double2 *sb = shift + (int64_t)(oct ? oct[c] : 0) * NC2 * h2 + m;
            double2 t[CI2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) t[k2] = __ldg(&sb[(int64_t)(g + CI1 * k2) * h2]);
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_mul(x[k2], t[k2]);
          }
          if (c != c0) {
            double2 t[CI2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) t[k2] = ob[(int64_t)(g + CI1 * k2) * h2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_add(x[k2], t[k2]);
          }
#pragma unroll
          for (int k2 = 0; k2 < CI2; ++k2) ob[(int64_t)(g + CI1 * k2) * h2] = x[k2];
        }
      }
    }
  }
}

// Single-pass downward resample (anterpolation / L2L): per child c, the columns of
// conj(shift[oct[c]]) * in[par[c]] (nth -> nth2, steps 1-3) into a shared [nth2][nph/2]
// intermediate, then the rows n <= nth2/2 (steps 4-5, nph -> nph2) back to half storage (+ add).
template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
__global__ void __launch_bounds__(128) box2_down_kernel(const double2 *__restrict__ in, int64_t nitem,
                                                       const int32_t *__restrict__ par,
                                                       const int8_t *__restrict__ oct,
                                                       const double2 *__restrict__ shift,
                                                       const double2 *__restrict__ twR, const double2 *__restrict__ twR2,
                                                       const double2 *__restrict__ twC, const double2 *__restrict__ twC2,
                                                       const double2 *__restrict__ add, double2 *__restrict__ out) {
  constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2;   // nph -> nph2 (rows)
  constexpr int NC = CF1 * CF2, NC2 = CI1 * CI2;   // nth -> nth2 (columns)
  using BC = Box2Cols<CF1, CF2, CI1, CI2>;
  constexpr int h = NR / 2, h2 = NR2 / 2, nrow = NC2 / 2 + 1;
  constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  constexpr int VW = 32 / G;
  constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  constexpr int IP = h + 1;                        // intermediate [NC2][IP]
  constexpr int KR = ((NR < NR2 ? NR : NR2) - 1) / 2, KC = ((NC < NC2 ? NC : NC2) - 1) / 2;
  extern __shared__ double2 sm[];
  double2 *tr1 = sm, *tr2 = tr1 + NR, *tc1 = tr2 + NR2, *tc2 = tc1 + NC;
  double2 *inter = tc2 + NC2;
  double2 *rbuf = inter + NC2 * IP;
  double2 *cbuf = rbuf + 4 * VW * RBUF;
  for (int j = threadIdx.x; j < NR; j += blockDim.x) tr1[j] = twR[j];
  for (int j = threadIdx.x; j < NR2; j += blockDim.x) tr2[j] = twR2[j];
  for (int j = threadIdx.x; j < NC; j += blockDim.x) tc1[j] = twC[j];
  for (int j = threadIdx.x; j < NC2; j += blockDim.x) tc2[j] = twC2[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, gr = lane - grp * G;
  double2 *rb = rbuf + (warp * VW + grp) * RBUF;
  const int v = threadIdx.x % BC::CW, g = threadIdx.x / BC::CW;
  for (int64_t c = blockIdx.x; c < nitem; c += gridDim.x) {
    double2 x[16];
    const double2 *pb = in + (int64_t)(par ? par[c] : c) * NC * h;
    const double2 *sbase = shift ? shift + (int64_t)(oct ? oct[c] : 0) * NC * h : nullptr;
    // ---- columns m < h of the shifted parent: nth -> nth2 into inter[t][m] ----
    for (int m0 = 0; m0 < h; m0 += BC::CW) {
      const int m = m0 + v;
      const bool mok = m < h;
      __syncthreads();
      if (g < CF2) {
#pragma unroll
        for (int n1 = 0; n1 < CF1; ++n1) x[n1] = mok ? pb[(CF2 * n1 + g) * h + m] : make_double2(0.0, 0.0);
        if (sbase && mok) {
          double2 t[CF1];
#pragma unroll
          for (int n1 = 0; n1 < CF1; ++n1) t[n1] = __ldg(&sbase[(CF2 * n1 + g) * h + m]);
#pragma unroll
          for (int n1 = 0; n1 < CF1; ++n1) x[n1] = c_mul(x[n1], c_conj(t[n1]));
        }
        dft<CF1>(x);
#pragma unroll
        for (int k1 = 1; k1 < CF1; ++k1) x[k1] = c_mul(x[k1], tc1[g * k1]);
#pragma unroll
        for (int k1 = 0; k1 < CF1; ++k1) cbuf[(k1 * (CF2 + 1) + g) * BC::CWP + v] = x[k1];
      }
      __syncthreads();
      if (g < CF1) {
#pragma unroll
        for (int n2 = 0; n2 < CF2; ++n2) x[n2] = cbuf[(g * (CF2 + 1) + n2) * BC::CWP + v];
      }
      __syncthreads();
      if (g < CF1) {
        dft<CF2>(x);
#pragma unroll
        for (int k2 = 0; k2 < CF2; ++k2) cbuf[(g + CF1 * k2) * BC::CWP + v] = x[k2];
      }
      __syncthreads();
      if (g < CI2) {
#pragma unroll
        for (int m1 = 0; m1 < CI1; ++m1) {
          const int i = CI2 * m1 + g;
          const int f = (i <= NC2 / 2) ? i : i - NC2;
          double2 z = make_double2(0.0, 0.0);
          if (f <= KC && f >= -KC) {
            const double2 y = cbuf[(f >= 0 ? f : f + NC) * BC::CWP + v];
            z = make_double2(y.x * (1.0 / NC), -y.y * (1.0 / NC));
          }
          x[m1] = z;
        }
      }
      __syncthreads();
      if (g < CI2) {
        dft<CI1>(x);
#pragma unroll
        for (int k1 = 1; k1 < CI1; ++k1) x[k1] = c_mul(x[k1], tc2[g * k1]);
#pragma unroll
        for (int k1 = 0; k1 < CI1; ++k1) cbuf[(k1 * (CI2 + 1) + g) * BC::CWP + v] = x[k1];
      }
      __syncthreads();
      if (g < CI1 && mok) {
#pragma unroll
        for (int n2 = 0; n2 < CI2; ++n2) x[n2] = cbuf[(g * (CI2 + 1) + n2) * BC::CWP + v];
        dft<CI2>(x);
#pragma unroll
        for (int k2 = 0; k2 < CI2; ++k2) inter[(g + CI1 * k2) * IP + m] = c_conj(x[k2]);
      }
    }
    __syncthreads();
    // ---- rows n <= nth2/2: nph -> nph2, back to half storage of child c (+ add) ----
    for (int r0 = warp * VW; r0 < nrow; r0 += 4 * VW) {
      const int n = r0 + grp;
      const bool vok = n < nrow && grp < VW;
      if (vok && gr < RF2) {
        const double2 *lo = inter + n * IP, *hi = inter + (n == 0 ? 0 : NC2 - n) * IP;
#pragma unroll
        for (int n1 = 0; n1 < RF1; ++n1) {
          const int e = RF2 * n1 + gr;
          x[n1] = e < h ? lo[e] : hi[e - h];
        }
        dft<RF1>(x);
#pragma unroll
        for (int k1 = 1; k1 < RF1; ++k1) x[k1] = c_mul(x[k1], tr1[gr * k1]);
#pragma unroll
        for (int k1 = 0; k1 < RF1; ++k1) rb[k1 * (RF2 + 1) + gr] = x[k1];
      }
      __syncwarp();
      if (vok && gr < RF1) {
#pragma unroll
        for (int n2 = 0; n2 < RF2; ++n2) x[n2] = rb[gr * (RF2 + 1) + n2];
      }
      __syncwarp();
      if (vok && gr < RF1) {
        dft<RF2>(x);
#pragma unroll
        for (int k2 = 0; k2 < RF2; ++k2) rb[gr + RF1 * k2] = x[k2];
      }
      __syncwarp();
      if (vok && gr < RI2) {
#pragma unroll
        for (int m1 = 0; m1 < RI1; ++m1) {
          const int i = RI2 * m1 + gr;
          const int f = (i <= NR2 / 2) ? i : i - NR2;
          double2 z = make_double2(0.0, 0.0);
          if (f <= KR && f >= -KR) {
            const double2 y = rb[f >= 0 ? f : f + NR];
            z = make_double2(y.x * (1.0 / NR), -y.y * (1.0 / NR));
          }
          x[m1] = z;
        }
      }
      __syncwarp();
      if (vok && gr < RI2) {
        dft<RI1>(x);
#pragma unroll
        for (int k1 = 1; k1 < RI1; ++k1) x[k1] = c_mul(x[k1], tr2[gr * k1]);
#pragma unroll
        for (int k1 = 0; k1 < RI1; ++k1) rb[k1 * (RI2 + 1) + gr] = x[k1];
      }
      __syncwarp();
      if (vok && gr < RI1) {
#pragma unroll
        for (int n2 = 0; n2 < RI2; ++n2) x[n2] = rb[gr * (RI2 + 1) + n2];
        dft<RI2>(x);
        const bool mirror = !(n == 0 || 2 * n == NC2);
#pragma unroll
        for (int k2 = 0; k2 < RI2; ++k2) {
          const int t = gr + RI1 * k2;
          if (t >= h2 && !mirror) continue;  // both halves are the same points
          const int64_t o = (c * NC2 + (t < h2 ? n : NC2 - n)) * h2 + (t < h2 ? t : t - h2);
          double2 val = c_conj(x[k2]);
          if (add) val = c_add(val, add[o]);
          out[o] = val;
        }
      }
      __syncwarp();
    }
  }
}

template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
static void launch_box2d_t(const double2 *in, int64_t nitem, const int32_t *par, const int8_t *oct,
                           const double2 *shift, const double2 *add, double2 *out, const TwiddleSet &tw,
                           cudaStream_t s) {
  constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2, NC = CF1 * CF2, NC2 = CI1 * CI2;
  using BC = Box2Cols<CF1, CF2, CI1, CI2>;
  constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  const size_t smem = ((size_t)NR + NR2 + NC + NC2 + (size_t)NC2 * (NR / 2 + 1) + 4 * (32 / G) * RBUF +
                       (size_t)CBUF * BC::CWP) * sizeof(double2);
  auto kern = box2_down_kernel<RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nitem, (int64_t)nsm * std::max(per, 1)));
  kern<<<grid, 128, smem, s>>>(in, nitem, par, oct, shift, tw.d + tw.offset[NR], tw.d + tw.offset[NR2],
                               tw.d + tw.offset[NC], tw.d + tw.offset[NC2], add, out);
}

template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
static void launch_box2_t(const double2 *in, int64_t nitem, const int32_t *cbeg, int64_t cbase, const int8_t *oct,
                          const double2 *shift, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2, NC = CF1 * CF2, NC2 = CI1 * CI2;
  using BC = Box2Cols<CF1, CF2, CI1, CI2>;
  constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  const size_t smem = ((size_t)NR + NR2 + NC + NC2 + (size_t)(NC / 2 + 1) * (NR2 + 1) + 4 * (32 / G) * RBUF +
                       (size_t)CBUF * BC::CWP) * sizeof(double2);
  auto kern = box2_up_kernel<RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nitem, (int64_t)nsm * std::max(per, 1)));
  kern<<<grid, 128, smem, s>>>(in, nitem, cbeg, cbase, oct, shift, tw.d + tw.offset[NR], tw.d + tw.offset[NR2],
                               tw.d + tw.offset[NC], tw.d + tw.offset[NC2], out);
}

// (nth, nph) -> (nth2, nph2) upward resamples done in one pass (square grids of the C2 microbench
// B8 / B16 and the C4 translation-only levels); false: use the two-pass kernels
static bool box2_4090() {  // single pass for 40 <-> 90x96 (else the two-pass rs2 kernels; A/B)
  static const int v = [] {
    const char *e = getenv("HFMM_BOX2_4090");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

static bool box2_big() {  // single pass for 64 <-> 128 grids (A/B switch HFMM_BOX2_BIG)
  static const int v = [] {
    const char *e = getenv("HFMM_BOX2_BIG");
    return e ? atoi(e) : 0;
  }();
  return v != 0;
}

// Grids with a single-pass kernel, keyed by (nth, nph, nth2, nph2); the template factors are
// (rows nph -> nph2, columns nth -> nth2).  C2: B8 / B16 square grids; BASELINE matvec configs: the
// translation-only levels of C3 / C5 (28 <-> 40 <-> 54x56) and C4 (24 <-> 32 <-> 42x48 <-> 60).
static constexpr int64_t gkey(int a, int b, int c, int d) { return (((int64_t)a * 1000 + b) * 1000 + c) * 1000 + d; }

bool box2_up_applies(int nth, int nph, int nth2, int nph2) {
  if (!rs2_enabled()) return false;
  switch (gkey(nth, nph, nth2, nph2)) {
    case gkey(16, 16, 32, 32): case gkey(32, 32, 64, 64): case gkey(24, 24, 32, 32):
    case gkey(32, 32, 42, 48): case gkey(42, 48, 60, 60): case gkey(28, 28, 40, 40): case gkey(40, 40, 54, 56):
    case gkey(40, 40, 90, 96):
      return box2_4090();
    case gkey(64, 64, 128, 128): return box2_big();
    default: return false;
  }
}

bool box2_down_applies(int nth, int nph, int nth2, int nph2) {
  if (!rs2_enabled()) return false;
  switch (gkey(nth, nph, nth2, nph2)) {
    case gkey(32, 32, 16, 16): case gkey(64, 64, 32, 32): case gkey(32, 32, 24, 24):
    case gkey(42, 48, 32, 32): case gkey(60, 60, 42, 48): case gkey(40, 40, 28, 28): case gkey(54, 56, 40, 40):
    case gkey(90, 96, 40, 40):
      return box2_4090();
    case gkey(128, 128, 64, 64): return box2_big();
    default: return false;
  }
}

// downward single pass: child c = R(conj(shift[oct[c]]) * in[par[c]]) (+ add[c]), c < nitem
bool launch_box2_down(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *par,
                      const int8_t *oct, const double2 *shift, const double2 *add, double2 *out, const TwiddleSet &tw,
                      cudaStream_t s) {
  if (launch_sym2_down(in, nitem, nth, nph, nth2, nph2, par, oct, shift, add, out, tw, s)) return true;
  if (!box2_down_applies(nth, nph, nth2, nph2)) return false;
  switch (gkey(nth, nph, nth2, nph2)) {
#define B2D(a, b, c, d, R1, R2, R3, R4, C1, C2, C3, C4)                                                      \
  case gkey(a, b, c, d):                                                                                     \
    launch_box2d_t<R1, R2, R3, R4, C1, C2, C3, C4>(in, nitem, par, oct, shift, add, out, tw, s);            \
    return true;
    B2D(32, 32, 16, 16, 8, 4, 4, 4, 8, 4, 4, 4)
    B2D(64, 64, 32, 32, 8, 8, 8, 4, 8, 8, 8, 4)
    B2D(32, 32, 24, 24, 8, 4, 6, 4, 8, 4, 6, 4)
    B2D(128, 128, 64, 64, 16, 8, 8, 8, 16, 8, 8, 8)
    B2D(42, 48, 32, 32, 8, 6, 8, 4, 7, 6, 8, 4)
    B2D(60, 60, 42, 48, 10, 6, 8, 6, 10, 6, 7, 6)
    B2D(40, 40, 28, 28, 8, 5, 7, 4, 8, 5, 7, 4)
    B2D(54, 56, 40, 40, 8, 7, 8, 5, 9, 6, 8, 5)
    B2D(90, 96, 40, 40, 12, 8, 8, 5, 10, 9, 8, 5)
#undef B2D
    default: return false;
  }
}

bool launch_box2_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, const TwiddleSet &tw,
                    cudaStream_t s) {
  if (launch_sym2_up(in, nitem, nth, nph, nth2, nph2, cbeg, cbase, oct, shift, out, tw, s)) return true;
  if (!box2_up_applies(nth, nph, nth2, nph2)) return false;
  switch (gkey(nth, nph, nth2, nph2)) {
#define B2U(a, b, c, d, R1, R2, R3, R4, C1, C2, C3, C4)                                                      \
  case gkey(a, b, c, d):                                                                                     \
    launch_box2_t<R1, R2, R3, R4, C1, C2, C3, C4>(in, nitem, cbeg, cbase, oct, shift, out, tw, s);          \
    return true;
    B2U(16, 16, 32, 32, 4, 4, 8, 4, 4, 4, 8, 4)
    B2U(32, 32, 64, 64, 8, 4, 8, 8, 8, 4, 8, 8)
    B2U(24, 24, 32, 32, 6, 4, 8, 4, 6, 4, 8, 4)
    B2U(64, 64, 128, 128, 8, 8, 16, 8, 8, 8, 16, 8)
    B2U(32, 32, 42, 48, 8, 4, 8, 6, 8, 4, 7, 6)
    B2U(42, 48, 60, 60, 8, 6, 10, 6, 7, 6, 10, 6)
    B2U(28, 28, 40, 40, 7, 4, 8, 5, 7, 4, 8, 5)
    B2U(40, 40, 54, 56, 8, 5, 8, 7, 8, 5, 9, 6)
    B2U(40, 40, 90, 96, 8, 5, 12, 8, 8, 5, 10, 9)
#undef B2U
    default: return false;
  }
}

// Tile plan per size (A/B on the C2 sizes): grids of <= 128 points use radix <= 8 butterflies
// (~75 registers) in 48 KB tiles; larger grids radix-16 butterflies (~140 registers) in 72 KB tiles.
struct TilePlan {
  int maxr;
  size_t smem_budget;
};
#ifndef HFMM_RS_BIG_MAXR
#define HFMM_RS_BIG_MAXR 16
#endif
#ifndef HFMM_RS_BIG_KB
#define HFMM_RS_BIG_KB 72
#endif
#ifndef HFMM_RS_SMALL_KB
#define HFMM_RS_SMALL_KB 48
#endif
static TilePlan tile_plan(int maxn) {
  return maxn > 128 ? TilePlan{HFMM_RS_BIG_MAXR, (size_t)HFMM_RS_BIG_KB * 1024} : TilePlan{8, (size_t)HFMM_RS_SMALL_KB * 1024};
}

static void set_smem(const void *fn, size_t bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static int rows_per_cta(int pitch, size_t budget) {
  int RB = 1;
  while (RB < 128 && (size_t)(2 * 2 * RB) * pitch * sizeof(double2) <= budget) RB *= 2;
  return RB;
}
static int cols_per_cta(int maxn, int ncols, size_t budget) {
  int CB = 1;
  while (CB < 32 && CB < ncols && (size_t)2 * maxn * ((2 * CB) | 1) * sizeof(double2) <= budget) CB *= 2;
  return CB;
}

template <bool UP, int MAXR>
static void launch_rows_t(const double2 *in, int64_t nbox, int nth, int nph, int nph2, const double2 *add,
                          double2 *out, size_t budget, const TwiddleSet &tw, cudaStream_t s) {
  const int64_t total = nbox * (nth / 2 + 1);
  const int pitch = std::max(nph, nph2) | 1;
  const int RB = rows_per_cta(pitch, budget);
  const size_t smem = (size_t)2 * RB * pitch * sizeof(double2);
  set_smem((const void *)rows_kernel<UP, MAXR>, smem);
  rows_kernel<UP, MAXR><<<(unsigned)((total + RB - 1) / RB), RS_TPB, smem, s>>>(
      in, nbox, nth, nph, nph2, RB, pitch, rlen(tw, nph, MAXR), rlen(tw, nph2, MAXR), add, out);
}

template <bool UP>
static void launch_rows(const double2 *in, int64_t nbox, int nth, int nph, int nph2, const double2 *add,
                        double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (nbox * (nth / 2 + 1) <= 0) return;
  const TilePlan tp = tile_plan(std::max(nph, nph2));
  if (tp.maxr >= 16) launch_rows_t<UP, 16>(in, nbox, nth, nph, nph2, add, out, tp.smem_budget, tw, s);
  else launch_rows_t<UP, 8>(in, nbox, nth, nph, nph2, add, out, tp.smem_budget, tw, s);
}

template <bool UP, int MAXR>
static void launch_cols_t(const double2 *in, int64_t nitem, int nth, int ncols, int rowlen, int nth2,
                          const int32_t *cbeg, int64_t cbase, const int32_t *par, const int8_t *oct,
                          const double2 *shift, double2 *out, size_t budget, const TwiddleSet &tw, cudaStream_t s) {
  const int maxn = std::max(nth, nth2);
  const int CB = cols_per_cta(maxn, ncols, budget);
  const int cp = CB | 1;
  const size_t smem = (size_t)2 * maxn * cp * sizeof(double2);
  set_smem((const void *)cols_kernel<UP, MAXR>, smem);
  const int64_t nstrip = (ncols + CB - 1) / CB;
  cols_kernel<UP, MAXR><<<(unsigned)(nitem * nstrip), RS_COLS_TPB, smem, s>>>(
      in, nitem, nth, ncols, rowlen, nth2, CB, cp, cbeg, cbase, par, oct, shift, rlen(tw, nth, MAXR),
      rlen(tw, nth2, MAXR), out);
}

template <bool UP>
static void launch_cols(const double2 *in, int64_t nitem, int nth, int ncols, int rowlen, int nth2,
                        const int32_t *cbeg, int64_t cbase, const int32_t *par, const int8_t *oct,
                        const double2 *shift, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (nitem <= 0 || ncols <= 0) return;
  TilePlan tp = tile_plan(std::max(nth, nth2));
  if (HFMM_RS_COLS_KB > 0) tp.smem_budget = (size_t)HFMM_RS_COLS_KB * 1024;
  if (tp.maxr >= 16)
    launch_cols_t<UP, 16>(in, nitem, nth, ncols, rowlen, nth2, cbeg, cbase, par, oct, shift, out, tp.smem_budget, tw, s);
  else
    launch_cols_t<UP, 8>(in, nitem, nth, ncols, rowlen, nth2, cbeg, cbase, par, oct, shift, out, tp.smem_budget, tw, s);
}

void launch_rows_up(const double2 *in, int64_t nbox, int nth, int nph, int nph2, double2 *tmp,
                    const TwiddleSet &tw, cudaStream_t s) {
  if (launch_rows2<true>(in, nbox, nth, nph, nph2, nullptr, tmp, tw, s)) return;
  launch_rows<true>(in, nbox, nth, nph, nph2, nullptr, tmp, tw, s);
}

void launch_cols_up(const double2 *tmp, int nth, int nph2, int nth2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, int64_t nparent, const double2 *shift, double2 *out,
                    const TwiddleSet &tw, cudaStream_t s) {
  if (launch_cols2<true>(tmp, nparent, nth, nph2 / 2, nph2, nth2, cbeg, cbase, nullptr, oct, shift, out, tw, s))
    return;
  launch_cols<true>(tmp, nparent, nth, nph2 / 2, nph2, nth2, cbeg, cbase, nullptr, oct, shift, out, tw, s);
}

void launch_cols_down(const double2 *in, int nth, int nph, int nth2, const int32_t *par,
                      const int8_t *oct, int64_t nchild, const double2 *shift, double2 *tmp,
                      const TwiddleSet &tw, cudaStream_t s) {
  if (launch_cols2<false>(in, nchild, nth, nph / 2, nph / 2, nth2, nullptr, 0, par, oct, shift, tmp, tw, s)) return;
  launch_cols<false>(in, nchild, nth, nph / 2, nph / 2, nth2, nullptr, 0, par, oct, shift, tmp, tw, s);
}

void launch_rows_down(const double2 *tmp, int64_t nbox, int nth2, int nph, int nph2,
                      const double2 *add, double2 *out, const TwiddleSet &tw, cudaStream_t s) {
  if (launch_rows2<false>(tmp, nbox, nth2, nph, nph2, add, out, tw, s)) return;
  launch_rows<false>(tmp, nbox, nth2, nph, nph2, add, out, tw, s);
}

}  // namespace hfmm
