// Register-resident complex arithmetic and small DFTs shared by the FFT resampling kernels
// (kernels_fft.cu: 5-step passes; kernels_sym.cu: coefficient-domain symmetric resampling).
// Product code (sm_100a); nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>

namespace hfmm {

__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 c_mi(double2 a) { return make_double2(a.y, -a.x); }  // -i a

// ---- forward small DFTs in registers: out[t] = sum_s v[s] e^{-2 pi i s t / R} -------------------
__device__ __forceinline__ void dft4(double2 &a0, double2 &a1, double2 &a2, double2 &a3) {
  const double2 s0 = c_add(a0, a2), d0 = c_sub(a0, a2);
  const double2 s1 = c_add(a1, a3), d1 = c_mi(c_sub(a1, a3));
  a0 = c_add(s0, s1);
  a2 = c_sub(s0, s1);
  a1 = c_add(d0, d1);
  a3 = c_sub(d0, d1);
}

template <int R>
__device__ __forceinline__ void dft(double2 *v);

template <>
__device__ __forceinline__ void dft<2>(double2 *v) {
  const double2 a = v[0], b = v[1];
  v[0] = c_add(a, b);
  v[1] = c_sub(a, b);
}
template <>
__device__ __forceinline__ void dft<4>(double2 *v) {
  dft4(v[0], v[1], v[2], v[3]);
}
template <>
__device__ __forceinline__ void dft<3>(double2 *v) {
  const double c = -0.5, s = -0.86602540378443864676372317075294;  // e^{-2 pi i/3}
  const double2 t1 = c_add(v[1], v[2]), t2 = c_sub(v[1], v[2]);
  const double2 m1 = make_double2(fma(c, t1.x, v[0].x), fma(c, t1.y, v[0].y));
  const double2 m2 = make_double2(-s * t2.y, s * t2.x);
  v[0] = c_add(v[0], t1);
  v[1] = c_add(m1, m2);
  v[2] = c_sub(m1, m2);
}
template <int R>
__device__ __forceinline__ void dft_odd(double2 *v) {  // R = 5, 7: symmetric pairs
  constexpr int H = R / 2;
  double c[H], s[H];
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    c[k - 1] = (R == 5) ? (k == 1 ? 0.30901699437494742410 : -0.80901699437494742410)
                        : (k == 1 ? 0.62348980185873353053 : k == 2 ? -0.22252093395631440429 : -0.90096886790241912624);
    s[k - 1] = (R == 5) ? (k == 1 ? -0.95105651629515357212 : -0.58778525229247312917)
                        : (k == 1 ? -0.78183148246802980871 : k == 2 ? -0.97492791218182360702 : -0.43388373911755812048);
  }
  double2 a[H], b[H];
#pragma unroll
  for (int k = 1; k <= H; ++k) a[k - 1] = c_add(v[k], v[R - k]), b[k - 1] = c_sub(v[k], v[R - k]);
  double2 o[R];
  double2 s0 = v[0];
#pragma unroll
  for (int k = 0; k < H; ++k) s0 = c_add(s0, a[k]);
  o[0] = s0;
#pragma unroll
  for (int t = 1; t <= H; ++t) {
    double2 re = v[0], im = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      const int e = (k * t) % R;
      const int ee = e <= H ? e : R - e;
      const double cs = c[ee - 1];
      const double sn = e <= H ? s[ee - 1] : -s[ee - 1];
      re = make_double2(fma(cs, a[k - 1].x, re.x), fma(cs, a[k - 1].y, re.y));
      im = make_double2(fma(sn, b[k - 1].x, im.x), fma(sn, b[k - 1].y, im.y));
    }
    // X_t = re + i im, X_{R-t} = re - i im
    o[t] = make_double2(re.x - im.y, re.y + im.x);
    o[R - t] = make_double2(re.x + im.y, re.y - im.x);
  }
#pragma unroll
  for (int t = 0; t < R; ++t) v[t] = o[t];
}
template <>
__device__ __forceinline__ void dft<5>(double2 *v) {
  dft_odd<5>(v);
}
template <>
__device__ __forceinline__ void dft<7>(double2 *v) {
  dft_odd<7>(v);
}
template <>
__device__ __forceinline__ void dft<8>(double2 *v) {
  const double h = 0.70710678118654752440;
  dft4(v[0], v[2], v[4], v[6]);
  dft4(v[1], v[3], v[5], v[7]);
  // odd part twiddles w8^k, k = 0..3
  const double2 o1 = make_double2(h * (v[3].x + v[3].y), h * (v[3].y - v[3].x));     // (1 - i)/sqrt2
  const double2 o2 = c_mi(v[5]);                                                     // -i
  const double2 o3 = make_double2(h * (v[7].y - v[7].x), -h * (v[7].x + v[7].y));    // (-1 - i)/sqrt2
  const double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1];
  v[0] = c_add(e0, o0);
  v[4] = c_sub(e0, o0);
  v[1] = c_add(e1, o1);
  v[5] = c_sub(e1, o1);
  v[2] = c_add(e2, o2);
  v[6] = c_sub(e2, o2);
  v[3] = c_add(e3, o3);
  v[7] = c_sub(e3, o3);
}
template <>
__device__ __forceinline__ void dft<16>(double2 *v) {
  // 16 = 4 x 4: DFT4 over q (stride 4), twiddle w16^{q k}, DFT4 over k
  dft4(v[0], v[4], v[8], v[12]);
  dft4(v[1], v[5], v[9], v[13]);
  dft4(v[2], v[6], v[10], v[14]);
  dft4(v[3], v[7], v[11], v[15]);
  // A_q[k] sits at v[q + 4 k]; multiply by w16^{q k}
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
  const double2 w1 = make_double2(c1, -s1), w2 = make_double2(h, -h), w3 = make_double2(s1, -c1);
  const double2 w6 = make_double2(-h, -h), w9 = make_double2(-c1, s1);
  v[5] = c_mul(v[5], w1);
  v[9] = c_mul(v[9], w2);
  v[13] = c_mul(v[13], w3);
  v[6] = c_mul(v[6], w2);
  v[10] = c_mi(v[10]);
  v[14] = c_mul(v[14], w6);
  v[7] = c_mul(v[7], w3);
  v[11] = c_mul(v[11], w6);
  v[15] = c_mul(v[15], w9);
  // X[k + 4 p] = sum_q A_q[k] w4^{q p}
  dft4(v[0], v[1], v[2], v[3]);
  dft4(v[4], v[5], v[6], v[7]);
  dft4(v[8], v[9], v[10], v[11]);
  dft4(v[12], v[13], v[14], v[15]);
  double2 o[16];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int p = 0; p < 4; ++p) o[k + 4 * p] = v[4 * k + p];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = o[t];
}

// ---- composite small DFTs N = P Q in registers (Cooley-Tukey, twiddles folded at compile time) ---
constexpr double kPiC = 3.14159265358979323846264338327950288;
__host__ __device__ constexpr double ct_sin(double x) {
  double t = x, s = x;
  for (int i = 1; i < 16; ++i) t *= -x * x / ((2.0 * i) * (2.0 * i + 1)), s += t;
  return s;
}
__host__ __device__ constexpr double ct_cos(double x) {
  double t = 1, s = 1;
  for (int i = 1; i < 16; ++i) t *= -x * x / ((2.0 * i - 1) * (2.0 * i)), s += t;
  return s;
}
// cos / sin of 2 pi K / N (argument reduced to [0, pi/2]; constant-folded when K, N are)
__host__ __device__ constexpr double cx_cos(int K, int N) {
  K %= N;
  double a = 2 * kPiC * K / N;
  if (a > kPiC) a -= 2 * kPiC;
  const double b = a < 0 ? -a : a;
  return b <= kPiC / 2 ? ct_cos(b) : -ct_cos(kPiC - b);
}
__host__ __device__ constexpr double cx_sin(int K, int N) {
  K %= N;
  double a = 2 * kPiC * K / N;
  if (a > kPiC) a -= 2 * kPiC;
  const double b = a < 0 ? -a : a;
  const double sb = b <= kPiC / 2 ? ct_sin(b) : ct_sin(kPiC - b);
  return a < 0 ? -sb : sb;
}
template <int P, int Q>
__device__ __forceinline__ void dft_pq(double2 *v) {  // X[k1 + P k2], n = Q n1 + n2
  constexpr int N = P * Q;
  double2 t[N];
#pragma unroll
  for (int n2 = 0; n2 < Q; ++n2) {
    double2 a[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) a[n1] = v[Q * n1 + n2];
    dft<P>(a);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1)
      t[n2 * P + k1] = (n2 * k1 == 0) ? a[k1]
                                      : c_mul(a[k1], make_double2(cx_cos(n2 * k1, N), -cx_sin(n2 * k1, N)));
  }
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) {
    double2 b[Q];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) b[n2] = t[n2 * P + k1];
    dft<Q>(b);
#pragma unroll
    for (int k2 = 0; k2 < Q; ++k2) v[k1 + P * k2] = b[k2];
  }
}
template <>
__device__ __forceinline__ void dft<1>(double2 *) {}
template <>
__device__ __forceinline__ void dft<6>(double2 *v) { dft_pq<3, 2>(v); }
template <>
__device__ __forceinline__ void dft<9>(double2 *v) { dft_pq<3, 3>(v); }
template <>
__device__ __forceinline__ void dft<10>(double2 *v) { dft_pq<5, 2>(v); }
template <>
__device__ __forceinline__ void dft<12>(double2 *v) { dft_pq<4, 3>(v); }
template <>
__device__ __forceinline__ void dft<14>(double2 *v) { dft_pq<7, 2>(v); }
template <>
__device__ __forceinline__ void dft<15>(double2 *v) { dft_pq<5, 3>(v); }


template <int A, int B>
struct Max2 {
  static constexpr int v = A > B ? A : B;
};

}  // namespace hfmm
