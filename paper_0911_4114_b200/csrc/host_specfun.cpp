// Host special functions for the plan (product code).
// j_n, y_n, h_n = j_n + i y_n (notation table); J_n enters through the Jacobi-Anger
// plane-wave spectrum eqn:PlaneWaveSpec used by Algs. 2-3.
#include <cmath>
#include <vector>

#include "hfmm_impl.h"

namespace hfmm {

static int miller_top(int nmax, double x) {
  double m = std::max((double)nmax, x);
  return (int)(m + 24.0 + 10.0 * std::cbrt(std::max(m, 1.0)));
}

// Downward recurrence j_{n-1} = (2n+1)/x j_n - j_{n+1}; scale fixed by the closed form of
// j_0 = sin x / x or j_1 = sin x / x^2 - cos x / x, whichever is larger in magnitude.
void sph_bessel_j(int nmax, double x, std::vector<double> &out) {
  int top = miller_top(nmax, x);
  std::vector<double> f(top + 2, 0.0);
  f[top] = 1.0;
  for (int n = top; n >= 1; --n) {
    f[n - 1] = (2.0 * n + 1.0) / x * f[n] - f[n + 1];
    if (std::fabs(f[n - 1]) > 1e150)
      for (int k = n - 1; k <= top; ++k) f[k] *= 1e-150;
  }
  double j0 = std::sin(x) / x;
  double j1 = std::sin(x) / (x * x) - std::cos(x) / x;
  double s = (std::fabs(j0) >= std::fabs(j1)) ? j0 / f[0] : j1 / f[1];
  out.assign(nmax + 1, 0.0);
  for (int n = 0; n <= nmax; ++n) out[n] = f[n] * s;
}

// Upward recurrence y_{n+1} = (2n+1)/x y_n - y_{n-1} (dominant solution, stable upward).
void sph_bessel_y(int nmax, double x, std::vector<double> &out) {
  out.assign(nmax + 1, 0.0);
  out[0] = -std::cos(x) / x;
  if (nmax >= 1) out[1] = -std::cos(x) / (x * x) - std::sin(x) / x;
  for (int n = 1; n < nmax; ++n) out[n + 1] = (2.0 * n + 1.0) / x * out[n] - out[n - 1];
}

// Cylindrical J_n: downward J_{n-1} = (2n/x) J_n - J_{n+1}, normalised by J_0 + 2 sum J_2k = 1.
void cyl_bessel_J(int nmax, double x, std::vector<double> &out) {
  out.assign(nmax + 1, 0.0);
  if (x == 0.0) {
    out[0] = 1.0;
    return;
  }
  int top = miller_top(nmax, x);
  top += top & 1;
  std::vector<double> f(top + 2, 0.0);
  f[top] = 1.0;
  for (int n = top; n >= 1; --n) {
    f[n - 1] = (2.0 * n) / x * f[n] - f[n + 1];
    if (std::fabs(f[n - 1]) > 1e150)
      for (int k = n - 1; k <= top; ++k) f[k] *= 1e-150;
  }
  double norm = f[0];
  for (int k = 2; k <= top; k += 2) norm += 2.0 * f[k];
  for (int n = 0; n <= nmax; ++n) out[n] = f[n] / norm;
}

}  // namespace hfmm
