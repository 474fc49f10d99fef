// Host-side plan of one level (product code): ell, N_theta, N_phi.
//   P:692-701  design radii |r0| = 2 a, |r| = alpha sqrt(3) a
//   P:146-165  ell from the EBF guess refined by the Carayol-Collino closed form
//   P:596-635  Alg. 2 (N_theta), eqn:EpsITheta, M(N, n) of P:613-619
//   P:637-686  Alg. 3 (N_phi(theta_n)), eqn:EpsIPhi
//   P:508-530  Alg. 1, one phi column at a time (the paper's own loop structure)
// Readings shared with DESIGN.md: threshold eps/(4 pi^2) in both searches; sizes restricted
// to 7-smooth values (N_theta even, N_phi multiple of 4; rectangular N_phi = smallest
// candidate at which every row n <= N_theta/2 passes); N^max = 4 ell + 64, doubled on failure.
#include <algorithm>
#include <cmath>
#include <vector>

#include "hfmm_impl.h"
#include "../../include/hfmm.h"

namespace hfmm {

static const double kPi = 3.14159265358979323846;

bool seven_smooth(int n) {
  if (n <= 0) return false;
  for (int p : {2, 3, 5, 7})
    while (n % p == 0) n /= p;
  return n == 1;
}

void transfer_series(int ell, double kappa, double r0norm, std::vector<cplx> &c) {
  std::vector<double> j, y;
  double x = kappa * r0norm;
  sph_bessel_j(ell, x, j);
  sph_bessel_y(ell, x, y);
  c.resize(ell + 1);
  cplx ipow(1.0, 0.0);
  const cplx pre(0.0, kappa / (4.0 * kPi));  // i kappa / (4 pi)
  for (int n = 0; n <= ell; ++n) {
    c[n] = pre * ipow * (2.0 * n + 1.0) * cplx(j[n], y[n]);
    ipow *= cplx(0.0, 1.0);
  }
}

static inline double sin_spectrum(int n) {  // F_n[|sin theta|]
  if (n & 1) return 0.0;
  return 2.0 / (kPi * (1.0 - (double)n * (double)n));
}

static inline cplx legendre_sum(const std::vector<cplx> &c, double t) {
  double p0 = 1.0, p1 = t;
  cplx acc = c[0];
  if (c.size() > 1) acc += c[1] * p1;
  for (size_t n = 1; n + 1 < c.size(); ++n) {
    double p2 = ((2.0 * n + 1.0) * t * p1 - (double)n * p0) / (double)(n + 1);
    acc += c[n + 1] * p2;
    p0 = p1;
    p1 = p2;
  }
  return acc;
}

// theta-spectrum (T^s)~_n, |n| <= nth/2 - 1, of one phi column (Alg. 1 lines 3-6)
static void alg1_spectrum(int ell, const std::vector<cplx> &c, const double r0hat[3], double phi,
                          int nth, std::vector<cplx> &ts) {
  const int P = 2 * ell + 1;
  std::vector<cplx> samp(P), tt(P);
  const double cp = std::cos(phi), sp = std::sin(phi);
  for (int j = 0; j < P; ++j) {
    double th = 2.0 * kPi * j / P;
    double st = std::sin(th), ct = std::cos(th);
    double t = cp * st * r0hat[0] + sp * st * r0hat[1] + ct * r0hat[2];
    t = std::max(-1.0, std::min(1.0, t));
    samp[j] = 0.5 * legendre_sum(c, t);
  }
  for (int f = -ell; f <= ell; ++f) {
    cplx acc = 0.0;
    for (int j = 0; j < P; ++j) {
      long long m = ((long long)f * j) % P;
      if (m < 0) m += P;
      double ang = -2.0 * kPi * (double)m / P;
      acc += samp[j] * cplx(std::cos(ang), std::sin(ang));
    }
    tt[f + ell] = acc / (double)P;
  }
  const int nb = nth / 2 - 1;
  ts.assign(2 * nb + 1, 0.0);
  for (int n = -nb; n <= nb; ++n) {
    cplx acc = 0.0;
    for (int f = -ell; f <= ell; ++f) acc += tt[f + ell] * sin_spectrum(n - f);
    ts[n + nb] = acc;
  }
}

void alg1_column(int ell, const std::vector<cplx> &c, const double r0hat[3], double phi,
                 int nth, std::vector<cplx> &out) {
  std::vector<cplx> ts;
  alg1_spectrum(ell, c, r0hat, phi, nth, ts);
  const int nb = nth / 2 - 1;
  out.assign(nth, 0.0);
  for (int p = 0; p < nth; ++p) {
    cplx acc = 0.0;
    for (int n = -nb; n <= nb; ++n) {
      long long m = ((long long)n * p) % nth;
      if (m < 0) m += nth;
      double ang = 2.0 * kPi * (double)m / nth;
      acc += ts[n + nb] * cplx(std::cos(ang), std::sin(ang));
    }
    out[p] = acc;
  }
}

double collino_bound(int ell, double kappa, double r, double r0) {
  std::vector<double> jr, jr0, yr0;
  sph_bessel_j(ell + 1, kappa * r, jr);
  sph_bessel_j(ell + 1, kappa * r0, jr0);
  sph_bessel_y(ell + 1, kappa * r0, yr0);
  cplx h1(jr0[ell + 1], yr0[ell + 1]), h0(jr0[ell], yr0[ell]);
  double best = 0.0;
  for (int s = 1; s >= -1; s -= 2) {
    double v = kappa * kappa * (r * r0 / (r0 + s * r)) * std::abs(h1 * jr[ell] + (double)s * h0 * jr[ell + 1]);
    if (!std::isfinite(v)) return INFINITY;
    best = std::max(best, v);
  }
  return best;
}

int select_ell(double kappa, double r, double r0, double eps, int *ell) {
  const double kr = kappa * r;
  if (kr <= 1.0) {  // EBF alone (reading R-2)
    double d0 = -std::log10(eps);
    *ell = std::max(1, (int)std::ceil(kr + 1.8 * std::pow(d0, 2.0 / 3.0) * std::cbrt(kr)));
    return 0;
  }
  int lo = std::max(1, (int)std::ceil(kr));
  // precompute j_n(kappa r), h_n(kappa r0) over a window and scan upward
  for (int span = 256; span <= 8192; span *= 2) {
    int nmax = lo + span + 1;
    std::vector<double> jr, jr0, yr0;
    sph_bessel_j(nmax, kr, jr);
    sph_bessel_j(nmax, kappa * r0, jr0);
    sph_bessel_y(nmax, kappa * r0, yr0);
    for (int l = lo; l < nmax; ++l) {
      cplx h1(jr0[l + 1], yr0[l + 1]), h0(jr0[l], yr0[l]);
      double best = 0.0;
      bool bad = false;
      for (int s = 1; s >= -1; s -= 2) {
        double v = kappa * kappa * (r * r0 / (r0 + s * r)) * std::abs(h1 * jr[l] + (double)s * h0 * jr[l + 1]);
        if (!std::isfinite(v)) bad = true;
        best = std::max(best, v);
      }
      if (bad) return HFMM_E_SEARCH;
      if (best < eps) {
        *ell = l;
        return 0;
      }
    }
  }
  return HFMM_E_SEARCH;
}

static inline int Mfun(int N, int n) {  // M(N, n)
  int a = n < 0 ? -n : n;
  return (2 * a < N) ? N - a : a;
}

int select_ntheta(int ell, double kappa, double r, double r0, double eps, int *nth) {
  const double thr = eps / (4.0 * kPi * kPi);
  std::vector<cplx> c;
  transfer_series(ell, kappa, r0, c);
  const double zhat[3] = {0.0, 0.0, 1.0};
  for (int nmax = 4 * ell + 64; nmax <= 64 * ell + 1024; nmax *= 2) {
    std::vector<cplx> ts;  // exact coefficients of T^{s,L} along z (Alg. 2 lines 2-3)
    alg1_spectrum(ell, c, zhat, 0.0, nmax, ts);
    const int nb = nmax / 2 - 1;
    std::vector<double> J;
    cyl_bessel_J(2 * nmax + 2, kappa * r, J);
    for (int N = 2 * ell; N < nmax; N += 2) {
      if (!seven_smooth(N)) continue;
      double bound = 0.0;
      for (int n = -nb; n <= nb; ++n) bound += std::abs(ts[n + nb]) * std::fabs(J[Mfun(N, n)]);
      if (bound < thr) {
        *nth = N;
        return 0;
      }
    }
  }
  return HFMM_E_SEARCH;
}

int select_nphi(int ell, double kappa, double r, double r0, double eps, int nth, int *nph,
                std::vector<int> *ragged, std::vector<int> *first7) {
  const double thr = eps / (4.0 * kPi * kPi);
  std::vector<cplx> c;
  transfer_series(ell, kappa, r0, c);
  const double xhat[3] = {1.0, 0.0, 0.0};
  const int P = 2 * ell + 1;
  const int rows = nth / 2 + 1;
  // T^{s,L}_{|r0| x}(theta_n, 2 pi m / (2l+1)) for rows n <= N_theta/2 (Alg. 3 line 3)
  std::vector<cplx> grid((size_t)rows * P);
#pragma omp parallel for schedule(dynamic)
  for (int m = 0; m < P; ++m) {
    std::vector<cplx> col;
    alg1_column(ell, c, xhat, 2.0 * kPi * m / P, nth, col);
    for (int n = 0; n < rows; ++n) grid[(size_t)n * P + m] = col[n];
  }
  int nmaxphi = 4 * ell + 64;
  nmaxphi -= nmaxphi % 4;
  std::vector<int> cands;
  for (int N = 4; N <= nmaxphi; N += 4) cands.push_back(N);
  std::vector<char> all_ok(cands.size(), 1);
  if (ragged) ragged->assign(rows, 0);
  if (first7) first7->assign(rows, -1);
  for (int n = 0; n < rows; ++n) {
    std::vector<double> tt(P);
    for (int f = -ell; f <= ell; ++f) {  // |F_m[T]| (Alg. 3 line 4)
      cplx acc = 0.0;
      for (int m = 0; m < P; ++m) {
        long long e = ((long long)f * m) % P;
        if (e < 0) e += P;
        double ang = -2.0 * kPi * (double)e / P;
        acc += grid[(size_t)n * P + m] * cplx(std::cos(ang), std::sin(ang));
      }
      tt[f + ell] = std::abs(acc) / (double)P;
    }
    double th = 2.0 * kPi * n / nth;
    std::vector<double> J;
    cyl_bessel_J(2 * nmaxphi + 2, kappa * r * std::fabs(std::sin(th)), J);
    int first = 0;
    for (size_t ci = 0; ci < cands.size(); ++ci) {
      int N = cands[ci];
      double bound = 0.0;
      for (int f = -ell; f <= ell; ++f) bound += tt[f + ell] * std::fabs(J[Mfun(N, f)]);
      bool ok = bound < thr;
      if (ok && !first) first = N;
      if (ok && first7 && (*first7)[n] < 0 && seven_smooth(N)) (*first7)[n] = N;
      if (!ok) all_ok[ci] = 0;
    }
    if (!first) return HFMM_E_SEARCH;
    if (ragged) (*ragged)[n] = first;
  }
  for (size_t ci = 0; ci < cands.size(); ++ci)
    if (all_ok[ci] && seven_smooth(cands[ci])) {
      *nph = cands[ci];
      return 0;
    }
  return HFMM_E_SEARCH;
}

// Ragged quadrature (R-15): N_phi(theta_n) = the smallest 7-smooth multiple of 4 at
// which row n passes Alg. 3's test at the level's final N_theta, capped at the rectangular N_phi;
// rows n > N_theta/2 mirror N_theta - n.
int select_nphi_rows(int ell, double kappa, double r, double r0, double eps, int nth, int cap,
                     std::vector<int> &rows) {
  int nph = 0;
  std::vector<int> f7;
  int rc = select_nphi(ell, kappa, r, r0, eps, nth, &nph, nullptr, &f7);
  if (rc) return rc;
  std::vector<int> half(nth / 2 + 1);
  for (int n = 0; n <= nth / 2; ++n) half[n] = (f7[n] > 0 && f7[n] <= cap) ? f7[n] : cap;
  std::vector<int> sym(half);  // exact theta -> pi - theta symmetry (rows n and N_theta/2 - n)
  for (int n = 0; n <= nth / 2; ++n) sym[n] = std::max(half[n], half[nth / 2 - n]);
  rows.assign(nth, cap);
  for (int n = 0; n < nth; ++n) rows[n] = sym[n <= nth / 2 ? n : nth - n];
  return 0;
}

// Translation-only level (R-14): the outgoing field of a box is a sum of plane waves
// e^{i kappa s.(x - c)}, |x - c| <= rho = (sqrt3/2) a, whose Fourier series in theta and in phi is
// the Jacobi-Anger series of eqn:PlaneWaveSpec with argument <= kappa rho.  Keeping
// |n| <= N/2 - 1 (R-6) drops 2 sum_{n >= N/2} |J_n(kappa rho)|; take the smallest even 7-smooth
// N_theta >= 4 and the smallest 7-smooth multiple of 4 N_phi with that tail <= eps / 100.
int select_rep_grid(double kappa, double a, double eps, int *nth, int *nph) {
  const double z = kappa * std::sqrt(3.0) / 2.0 * a, thr = eps * 1e-2;
  const int nmax = 4 * (int)std::ceil(z) + 256;
  std::vector<double> J;
  cyl_bessel_J(nmax + 40, z, J);
  std::vector<double> tail(nmax + 2, 0.0);  // tail[m] = 2 sum_{n >= m} |J_n|
  for (int m = nmax + 40; m >= nmax + 1; --m) tail[nmax + 1] += 2.0 * std::fabs(J[m]);
  for (int m = nmax; m >= 0; --m) tail[m] = tail[m + 1] + 2.0 * std::fabs(J[m]);
  *nth = *nph = 0;
  for (int N = 4; N <= 2 * nmax; N += 2)
    if (seven_smooth(N) && tail[N / 2] <= thr) {
      *nth = N;
      break;
    }
  for (int N = 4; N <= 2 * nmax; N += 4)
    if (seven_smooth(N) && tail[N / 2] <= thr) {
      *nph = N;
      break;
    }
  return (*nth && *nph) ? 0 : HFMM_E_SEARCH;
}

}  // namespace hfmm

extern "C" int hfmm_ragged_rows(double kappa, double a, double eps_level, double alpha, int ell, int n_theta,
                                int n_phi_cap, int *rows) {
  if (!(kappa > 0) || !(a > 0) || !(eps_level > 0) || !(alpha > 0) || ell < 1 || n_theta < 2 || n_phi_cap < 4 ||
      !rows)
    return HFMM_E_ARG;
  std::vector<int> r;
  int rc = hfmm::select_nphi_rows(ell, kappa, alpha * std::sqrt(3.0) * a, 2.0 * a, eps_level, n_theta, n_phi_cap, r);
  if (rc) return rc;
  for (int n = 0; n < n_theta; ++n) rows[n] = r[n];
  return 0;
}

extern "C" int hfmm_rep_grid(double kappa, double a, double eps, int *n_theta, int *n_phi) {
  if (!(kappa > 0) || !(a > 0) || !(eps > 0) || !n_theta || !n_phi) return HFMM_E_ARG;
  return hfmm::select_rep_grid(kappa, a, eps, n_theta, n_phi);
}

extern "C" int hfmm_level_quadrature(double kappa, double a, double eps_level, double alpha,
                                     int *ell, int *n_theta, int *n_phi, int *ragged,
                                     int ragged_cap) {
  using namespace hfmm;
  if (!(kappa > 0) || !(a > 0) || !(eps_level > 0) || !(alpha > 0) || alpha > 1 || !ell ||
      !n_theta || !n_phi)
    return HFMM_E_ARG;
  const double r = alpha * std::sqrt(3.0) * a, r0 = 2.0 * a;
  int rc = select_ell(kappa, r, r0, eps_level, ell);
  if (rc) return rc;
  rc = select_ntheta(*ell, kappa, r, r0, eps_level, n_theta);
  if (rc) return rc;
  std::vector<int> rg;
  rc = select_nphi(*ell, kappa, r, r0, eps_level, *n_theta, n_phi, &rg);
  if (rc) return rc;
  if (ragged)
    for (int i = 0; i < (int)rg.size() && i < ragged_cap; ++i) ragged[i] = rg[i];
  return 0;
}
