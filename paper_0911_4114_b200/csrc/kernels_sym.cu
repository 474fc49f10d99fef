// NEXT 4: coefficient-domain symmetric resampling (product code, sm_100a).
//
// The 5-step procedure (kernels_fft.cu) builds theta-periodic columns from phi SAMPLES
// with eqn:NumSphereSym.  P:749: "A slightly more efficient algorithm uses the symmetry
// eqn:FourierSphereSym", f~_{n,m} = (-1)^m f~_{-n,m}.  In the phi-coefficient domain:
// after the forward phi-DFT of the full rows n <= N_theta/2, the theta sequence of each
// phi-frequency m satisfies
//     c_m(theta_{N_theta - n}) = (-1)^m c_m(theta_n),
// i.e. it is even (m even) or odd (m odd) and known from n <= N_theta/2 alone; a band-limited
// theta resample keeps the parity.  So the sum h = c_e + c_o of an even-m and an odd-m sequence
// is resampled with ONE complex FFT pair and split afterwards,
//     c'_e(n) = (h'(n) + h'(-n)) / 2,      c'_o(n) = (h'(n) - h'(-n)) / 2,
// half the theta transforms of the sample-domain procedure; then the inverse phi-DFT of each
// output row n' <= N'_theta/2 gives the full row, stored to half storage (rows n', N'_theta - n').
// Same operator as the 5-step (bands |m| <= (min(N_phi, N'_phi) - 1)/2, |k| <= (min(N_theta,
// N'_theta) - 1)/2, R-6); parity vs oracle.resample in tests/test_gpu_next4.py.
//
// One CTA per item (the box2 layout of kernels_fft.cu): UP = parent with its children (rows of
// each child -> coefficients, pair columns, rows out x shift, summed over the children in the
// parent's output); DOWN = child c of parent par[c] (rows of conj(shift) * parent -> coefficients,
// pair columns, rows out + I_c).  The coefficient array [2 K_phi + 1][pitch] stays in shared memory.
// Opt-in (HFMM_NEXT4=1): the single-pass 5-step kernels stay the default (A/B in DESIGN.md).
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "hfmm_impl.h"
#include "fft_regs.cuh"

namespace hfmm {

constexpr int SYM_CW = 8, SYM_CWP = 9;   // column pairs per strip (lane & 7), exchange pitch

template <bool UP, int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
struct SymCfg {
  static constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2;    // phi: N_phi -> N'_phi (rows)
  static constexpr int NC = CF1 * CF2, NC2 = CI1 * CI2;    // theta: N_theta -> N'_theta (columns)
  static constexpr int h = NR / 2, h2 = NR2 / 2;
  static constexpr int nrow_in = NC / 2 + 1, nrow_out = NC2 / 2 + 1;
  static constexpr int KP = ((NR < NR2 ? NR : NR2) - 1) / 2;   // kept phi band
  static constexpr int KC = ((NC < NC2 ? NC : NC2) - 1) / 2;   // kept theta band
  static constexpr int NCOEF = 2 * KP + 1;
  static constexpr int PITCH = (Max2<nrow_in, nrow_out>::v) | 1;
  static constexpr int KE = (KP / 2) * 2, KO = (KP % 2) ? KP : KP - 1;  // largest even / odd <= KP
  static constexpr int NE = KE + 1, NO = KO + 1;                        // counts (step 2)
  static constexpr int NPAIR = NE > NO ? NE : NO;
  static constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  static constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  static constexpr int VW = 32 / G;
  static constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  static constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  static constexpr size_t smem_elems() {
    return (size_t)NR + NR2 + NC + NC2 + (size_t)NCOEF * PITCH + 4 * VW * RBUF + (size_t)CBUF * SYM_CWP;
  }
};

template <bool UP, int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
__global__ void __launch_bounds__(128) sym2_kernel(const double2 *__restrict__ in, int64_t nitem,
                                                  const int32_t *__restrict__ cbeg, int64_t cbase,
                                                  const int32_t *__restrict__ par, const int8_t *__restrict__ oct,
                                                  const double2 *__restrict__ shift,
                                                  const double2 *__restrict__ twR, const double2 *__restrict__ twR2,
                                                  const double2 *__restrict__ twC, const double2 *__restrict__ twC2,
                                                  const double2 *__restrict__ add, double2 *__restrict__ out) {
  using C = SymCfg<UP, RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  constexpr int NR = C::NR, NR2 = C::NR2, NC = C::NC, NC2 = C::NC2, h = C::h, h2 = C::h2;
  constexpr int KP = C::KP, KC = C::KC, P = C::PITCH, KE = C::KE, KO = C::KO, NE = C::NE, NO = C::NO;
  constexpr int G = C::G, VW = C::VW, RBUF = C::RBUF;
  extern __shared__ double2 sm[];
  double2 *tr1 = sm, *tr2 = tr1 + NR, *tc1 = tr2 + NR2, *tc2 = tc1 + NC;
  double2 *A = tc2 + NC2;                            // coefficients [NCOEF][P]: A[(m + KP) P + n]
  double2 *rbuf = A + C::NCOEF * P;                  // [4 warps][VW][RBUF]
  double2 *cbuf = rbuf + 4 * VW * RBUF;              // [CBUF][SYM_CWP]
  for (int j = threadIdx.x; j < NR; j += blockDim.x) tr1[j] = twR[j];
  for (int j = threadIdx.x; j < NR2; j += blockDim.x) tr2[j] = twR2[j];
  for (int j = threadIdx.x; j < NC; j += blockDim.x) tc1[j] = twC[j];
  for (int j = threadIdx.x; j < NC2; j += blockDim.x) tc2[j] = twC2[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, gr = lane - grp * G;     // row passes: lane group, lane in group
  double2 *rb = rbuf + (warp * VW + grp) * RBUF;
  const int v = threadIdx.x & (SYM_CW - 1), g = threadIdx.x >> 3;  // column pass: pair in strip, lane
  for (int64_t item = blockIdx.x; item < nitem; item += gridDim.x) {
    int64_t c0 = item, c1 = item + 1;
    if (UP && cbeg) c0 = cbeg[item], c1 = cbeg[item + 1];
    for (int64_t c = c0; c < c1; ++c) {
      double2 x[16];
      __syncthreads();  // twiddles staged / previous child's coefficients consumed
      // ---- (1) forward phi-DFT of the full rows n <= N_theta/2 -> A[m][n] (|m| <= KP, 1/N_phi) ----
      const double2 *src = UP ? in + (c - cbase) * (int64_t)NC * h : in + (int64_t)(par ? par[c] : c) * NC * h;
      const double2 *sh = (!UP && shift) ? shift + (int64_t)(oct ? oct[c] : 0) * NC * h : nullptr;
      for (int r0 = warp * VW; r0 < C::nrow_in; r0 += 4 * VW) {
        const int n = r0 + grp;
        const bool vok = n < C::nrow_in;
        const int nm = n == 0 ? 0 : NC - n;          // eqn:NumSphereSym partner row
        if (vok && gr < RF2) {
#pragma unroll
          for (int n1 = 0; n1 < RF1; ++n1) {
            const int e = RF2 * n1 + gr;
            const int64_t o = e < h ? (int64_t)n * h + e : (int64_t)nm * h + (e - h);
            double2 val = src[o];
            if (!UP && sh) val = c_mul(val, c_conj(__ldg(&sh[o])));   // L2L: conj shift on the parent grid
            x[n1] = val;
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
          dft<RF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < RF2; ++k2) {      // X[gr + RF1 k2]: frequency f
            const int f = gr + RF1 * k2;
            const int m = f <= NR / 2 ? f : f - NR;
            if (m <= KP && m >= -KP) A[(m + KP) * P + n] = make_double2(x[k2].x * (1.0 / NR), x[k2].y * (1.0 / NR));
          }
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- (2) theta resample of column pairs (even m_e, odd m_o): h = c_e + c_o over n < N_theta
      //      (eqn:FourierSphereSym), FFT N_theta, pad / truncate, inverse FFT N'_theta, split ----
      for (int j0 = 0; j0 < C::NPAIR; j0 += SYM_CW) {
        const int j = j0 + v;
        const bool has_e = j < NE, has_o = j < NO;
        const int me = -KE + 2 * j, mo = -KO + 2 * j;
        const double2 *ce = A + (has_e ? (me + KP) * P : 0), *co = A + (has_o ? (mo + KP) * P : 0);
        if (g < CF2) {
#pragma unroll
          for (int n1 = 0; n1 < CF1; ++n1) {
            const int n = CF2 * n1 + g;
            const bool low = 2 * n <= NC;
            const int nn = low ? n : NC - n;
            const double2 a = has_e ? ce[nn] : make_double2(0.0, 0.0);
            const double2 b = has_o ? co[nn] : make_double2(0.0, 0.0);
            x[n1] = low ? c_add(a, b) : c_sub(a, b);   // odd m: c(theta_{N - n}) = -c(theta_n)
          }
          dft<CF1>(x);
#pragma unroll
          for (int k1 = 1; k1 < CF1; ++k1) x[k1] = c_mul(x[k1], tc1[g * k1]);
#pragma unroll
          for (int k1 = 0; k1 < CF1; ++k1) cbuf[(k1 * (CF2 + 1) + g) * SYM_CWP + v] = x[k1];
        }
        __syncthreads();
        if (g < CF1) {
#pragma unroll
          for (int n2 = 0; n2 < CF2; ++n2) x[n2] = cbuf[(g * (CF2 + 1) + n2) * SYM_CWP + v];
        }
        __syncthreads();
        if (g < CF1) {
          dft<CF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < CF2; ++k2) cbuf[(g + CF1 * k2) * SYM_CWP + v] = x[k2];
        }
        __syncthreads();
        if (g < CI2) {  // padded / truncated conj spectrum (1/N_theta): Z[CI2 m1 + g]
#pragma unroll
          for (int m1 = 0; m1 < CI1; ++m1) {
            const int i = CI2 * m1 + g;
            const int f = (i <= NC2 / 2) ? i : i - NC2;
            double2 z = make_double2(0.0, 0.0);
            if (f <= KC && f >= -KC) {
              const double2 y = cbuf[(f >= 0 ? f : f + NC) * SYM_CWP + v];
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
          for (int k1 = 0; k1 < CI1; ++k1) cbuf[(k1 * (CI2 + 1) + g) * SYM_CWP + v] = x[k1];
        }
        __syncthreads();
        if (g < CI1) {
#pragma unroll
          for (int n2 = 0; n2 < CI2; ++n2) x[n2] = cbuf[(g * (CI2 + 1) + n2) * SYM_CWP + v];
          dft<CI2>(x);
        }
        __syncthreads();  // exchange buffer read: reuse it for h'(t), t < N'_theta
        if (g < CI1) {
#pragma unroll
          for (int k2 = 0; k2 < CI2; ++k2) cbuf[(g + CI1 * k2) * SYM_CWP + v] = c_conj(x[k2]);
        }
        __syncthreads();
        for (int n = g; n < C::nrow_out; n += 16) {   // split into the even / odd parts, n <= N'_theta/2
          const double2 hp = cbuf[n * SYM_CWP + v], hm = cbuf[((NC2 - n) % NC2) * SYM_CWP + v];
          if (has_e) A[(me + KP) * P + n] = make_double2(0.5 * (hp.x + hm.x), 0.5 * (hp.y + hm.y));
          if (has_o) A[(mo + KP) * P + n] = make_double2(0.5 * (hp.x - hm.x), 0.5 * (hp.y - hm.y));
        }
        __syncthreads();  // cbuf reused by the next strip
      }
      // ---- (3) inverse phi-DFT of the rows n' <= N'_theta/2 -> half storage (x shift / + I) ----
      for (int r0 = warp * VW; r0 < C::nrow_out; r0 += 4 * VW) {
        const int n = r0 + grp;
        const bool vok = n < C::nrow_out;
        if (vok && gr < RI2) {  // conj of the padded coefficient row: Z[RI2 m1 + gr]
#pragma unroll
          for (int m1 = 0; m1 < RI1; ++m1) {
            const int i = RI2 * m1 + gr;
            const int f = (i <= NR2 / 2) ? i : i - NR2;
            x[m1] = (f <= KP && f >= -KP) ? c_conj(A[(f + KP) * P + n]) : make_double2(0.0, 0.0);
          }
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
          const int64_t ob = (UP ? item : c) * (int64_t)NC2 * h2;
#pragma unroll
          for (int k2 = 0; k2 < RI2; ++k2) {
            const int t = gr + RI1 * k2;
            if (t >= h2 && !mirror) continue;     // both halves are the same points
            const int64_t o = (int64_t)(t < h2 ? n : NC2 - n) * h2 + (t < h2 ? t : t - h2);
            double2 val = c_conj(x[k2]);
            if (UP) {
              if (shift) val = c_mul(val, __ldg(&shift[(int64_t)(oct ? oct[c] : 0) * NC2 * h2 + o]));
              if (c != c0) val = c_add(val, out[ob + o]);
            } else if (add) {
              val = c_add(val, add[ob + o]);
            }
            out[ob + o] = val;
          }
        }
        __syncwarp();
      }
    }
  }
}

template <bool UP, int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
static void launch_sym2_t(const double2 *in, int64_t nitem, const int32_t *cbeg, int64_t cbase, const int32_t *par,
                          const int8_t *oct, const double2 *shift, const double2 *add, double2 *out,
                          const TwiddleSet &tw, cudaStream_t s) {
  using C = SymCfg<UP, RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  const size_t smem = C::smem_elems() * sizeof(double2);
  auto kern = sym2_kernel<UP, RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nitem, (int64_t)nsm * std::max(per, 1)));
  kern<<<grid, 128, smem, s>>>(in, nitem, cbeg, cbase, par, oct, shift, tw.d + tw.offset[C::NR],
                               tw.d + tw.offset[C::NR2], tw.d + tw.offset[C::NC], tw.d + tw.offset[C::NC2], add, out);
}

// Process-wide switch: HFMM_NEXT4 in the environment at load time, or hfmm_set_next4().
static std::atomic<int> g_next4{[] {
  const char *e = getenv("HFMM_NEXT4");
  return e ? atoi(e) : 0;
}()};

bool next4_enabled() { return g_next4.load(std::memory_order_relaxed) != 0; }

}  // namespace hfmm

extern "C" int hfmm_set_next4(int on) { return hfmm::g_next4.exchange(on ? 1 : 0); }

namespace hfmm {

static constexpr int64_t skey(int a, int b, int c, int d) { return (((int64_t)a * 1000 + b) * 1000 + c) * 1000 + d; }

// (nth, nph) -> (nth2, nph2); template factors (rows nph -> nph2, columns nth -> nth2)
#define SYM_UP_LIST(X)                                                \
  X(16, 16, 32, 32, 4, 4, 8, 4, 4, 4, 8, 4)                           \
  X(32, 32, 64, 64, 8, 4, 8, 8, 8, 4, 8, 8)                           \
  X(64, 64, 128, 128, 8, 8, 16, 8, 8, 8, 16, 8)                       \
  X(24, 24, 32, 32, 6, 4, 8, 4, 6, 4, 8, 4)                           \
  X(32, 32, 42, 48, 8, 4, 8, 6, 8, 4, 7, 6)                           \
  X(42, 48, 60, 60, 8, 6, 10, 6, 7, 6, 10, 6)                         \
  X(28, 28, 40, 40, 7, 4, 8, 5, 7, 4, 8, 5)                           \
  X(40, 40, 54, 56, 8, 5, 8, 7, 8, 5, 9, 6)
#define SYM_DOWN_LIST(X)                                              \
  X(32, 32, 16, 16, 8, 4, 4, 4, 8, 4, 4, 4)                           \
  X(64, 64, 32, 32, 8, 8, 8, 4, 8, 8, 8, 4)                           \
  X(128, 128, 64, 64, 16, 8, 8, 8, 16, 8, 8, 8)                       \
  X(32, 32, 24, 24, 8, 4, 6, 4, 8, 4, 6, 4)                           \
  X(42, 48, 32, 32, 8, 6, 8, 4, 7, 6, 8, 4)                           \
  X(60, 60, 42, 48, 10, 6, 8, 6, 10, 6, 7, 6)                         \
  X(40, 40, 28, 28, 8, 5, 7, 4, 8, 5, 7, 4)                           \
  X(54, 56, 40, 40, 8, 7, 8, 5, 9, 6, 8, 5)

bool sym2_up_applies(int nth, int nph, int nth2, int nph2) {
  if (!next4_enabled()) return false;
  switch (skey(nth, nph, nth2, nph2)) {
#define SYMA(a, b, c, d, ...) case skey(a, b, c, d): return true;
    SYM_UP_LIST(SYMA)
#undef SYMA
    default: return false;
  }
}

bool sym2_down_applies(int nth, int nph, int nth2, int nph2) {
  if (!next4_enabled()) return false;
  switch (skey(nth, nph, nth2, nph2)) {
#define SYMA(a, b, c, d, ...) case skey(a, b, c, d): return true;
    SYM_DOWN_LIST(SYMA)
#undef SYMA
    default: return false;
  }
}

bool launch_sym2_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, const TwiddleSet &tw,
                    cudaStream_t s) {
  if (!next4_enabled()) return false;
  switch (skey(nth, nph, nth2, nph2)) {
#define SYMU(a, b, c, d, R1, R2, R3, R4, C1, C2, C3, C4)                                               \
  case skey(a, b, c, d):                                                                               \
    launch_sym2_t<true, R1, R2, R3, R4, C1, C2, C3, C4>(in, nitem, cbeg, cbase, nullptr, oct, shift, nullptr, out, \
                                                       tw, s);                                        \
    return true;
    SYM_UP_LIST(SYMU)
#undef SYMU
    default: return false;
  }
}

bool launch_sym2_down(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *par,
                      const int8_t *oct, const double2 *shift, const double2 *add, double2 *out, const TwiddleSet &tw,
                      cudaStream_t s) {
  if (!next4_enabled()) return false;
  switch (skey(nth, nph, nth2, nph2)) {
#define SYMD(a, b, c, d, R1, R2, R3, R4, C1, C2, C3, C4)                                               \
  case skey(a, b, c, d):                                                                               \
    launch_sym2_t<false, R1, R2, R3, R4, C1, C2, C3, C4>(in, nitem, nullptr, 0, par, oct, shift, add, out, tw, s); \
    return true;
    SYM_DOWN_LIST(SYMD)
#undef SYMD
    default: return false;
  }
}

}  // namespace hfmm
