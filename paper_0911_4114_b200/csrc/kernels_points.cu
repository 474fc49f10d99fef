// Point-wise FP64 kernels of the matvec (product code, sm_100a):
//   P2P  near field, eqn:FMM_FinalStep second term
//   S2M  initialisation M^L_a(s) = sum psi_i e^{i kappa s.(x_i - c_a)}
//   L2T  field computation int L e^{i kappa s.(c_a - x_i)} dS
//   permute / combine (Morton order <-> caller order)
// All three main kernels are bound by the FP64 pipe (one complex exponential per pair or per
// (point, direction)); the exponential is computed by hfmm_cexpi() below: a 2-part Cody-Waite
// reduction by 2 pi / 256, a 256-entry table of e^{2 pi i t/256} in shared memory and
// short minimax-free Taylor polynomials on |r| <= pi/256 (|error| < 2 ulp).
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>

#include "hfmm_impl.h"

namespace hfmm {

#define HFMM_TABLE 256

// 2 pi / 256 split for Cody-Waite: hi has 24 significant bits (a float), so k * hi is exact
// for |k| < 2^29; lo = 2 pi / 256 - hi.
static constexpr double kInvStep = 40.743665431525205956834243423364;   // 256 / (2 pi)
static void step_split(double *hi, double *lo) {
  const double step = 6.283185307179586476925286766559 / 256.0;
  *hi = (double)(float)step;
  *lo = step - *hi;
}

// Exact e^{i 2 pi t / 256} table, filled once per block.
__device__ __forceinline__ void fill_exp_table(double2 *tab) {
  for (int t = threadIdx.x; t < HFMM_TABLE; t += blockDim.x) {
    double s, c;
    sincospi((double)t / (HFMM_TABLE / 2), &s, &c);
    tab[t] = make_double2(c, s);
  }
}

// e^{i x} for |x| < 2^20: x = k (2 pi / 256) + r, e^{ix} = tab[k mod 256] * e^{ir}
__device__ __forceinline__ double2 cexpi_tab(double x, const double2 *__restrict__ tab, double shi,
                                             double slo) {
  double kd = rint(x * kInvStep);
  double r = fma(-kd, shi, x);
  r = fma(-kd, slo, r);
  int k = ((int)kd) & (HFMM_TABLE - 1);
  double r2 = r * r;
  // sin r = r (1 - r^2/6 + r^4/120 - r^6/5040), cos r = 1 - r^2/2 + r^4/24 - r^6/720
  double sp = fma(r2, fma(r2, fma(r2, -1.0 / 5040.0, 1.0 / 120.0), -1.0 / 6.0), 1.0);
  double sr = r * sp;
  double cr = fma(r2, fma(r2, fma(r2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
  double2 e = tab[k];
  return make_double2(fma(e.x, cr, -e.y * sr), fma(e.x, sr, e.y * cr));
}

// ---------------------------------------------------------------------------------------------
// P2P: one thread per target, sources of every neighbour box streamed through shared memory.
// ---------------------------------------------------------------------------------------------
constexpr int P2P_TPB = 128;

__global__ void __launch_bounds__(P2P_TPB) p2p_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                      const int32_t *__restrict__ nb_row,
                                                      const int32_t *__restrict__ nb_box,
                                                      const int32_t *__restrict__ tile_leaf,
                                                      const int64_t *__restrict__ tile_begin,
                                                      double kappa, double shi, double slo,
                                                      double2 *__restrict__ y_near) {
  __shared__ double2 tab[HFMM_TABLE];
  __shared__ double sx[P2P_TPB], sy[P2P_TPB], sz[P2P_TPB];
  __shared__ double2 sq[P2P_TPB];
  fill_exp_table(tab);
  const int32_t leaf = tile_leaf[blockIdx.x];
  const int64_t t0 = tile_begin[blockIdx.x];
  const int64_t tend = first[leaf + 1];
  const int64_t i = t0 + threadIdx.x;
  const bool active = i < tend;
  const double xi = active ? pts.x[i] : 0.0, yi = active ? pts.y[i] : 0.0, zi = active ? pts.z[i] : 0.0;
  double ar = 0.0, ai = 0.0;
  for (int32_t e = nb_row[leaf]; e < nb_row[leaf + 1]; ++e) {
    const int32_t b = nb_box[e];
    const int64_t s0 = first[b], s1 = first[b + 1];
    for (int64_t c0 = s0; c0 < s1; c0 += P2P_TPB) {
      const int cnt = (int)min((int64_t)P2P_TPB, s1 - c0);
      __syncthreads();
      if (threadIdx.x < cnt) {
        const int64_t j = c0 + threadIdx.x;
        sx[threadIdx.x] = pts.x[j];
        sy[threadIdx.x] = pts.y[j];
        sz[threadIdx.x] = pts.z[j];
        sq[threadIdx.x] = pts.q[j];
      }
      __syncthreads();
#pragma unroll 4
      for (int u = 0; u < cnt; ++u) {
        const double dx = xi - sx[u], dy = yi - sy[u], dz = zi - sz[u];
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        const double rinv = (r2 > 0.0) ? rsqrt(r2) : 0.0;       // self pair excluded
        const double2 e = cexpi_tab(kappa * (r2 * rinv), tab, shi, slo);
        const double gr = e.x * rinv, gi = e.y * rinv;
        const double2 q = sq[u];
        ar = fma(gr, q.x, fma(-gi, q.y, ar));
        ai = fma(gr, q.y, fma(gi, q.x, ai));
      }
    }
  }
  if (active) y_near[i] = make_double2(ar, ai);
}

void launch_p2p(PointsDev pts, const int64_t *first, const int32_t *nb_row, const int32_t *nb_box,
                int32_t, int32_t, const int32_t *tile_leaf, const int64_t *tile_begin,
                int64_t ntiles, double kappa, double2 *y_near, cudaStream_t s) {
  if (ntiles <= 0) return;
  double shi, slo;
  step_split(&shi, &slo);
  p2p_kernel<<<(unsigned)ntiles, P2P_TPB, 0, s>>>(pts, first, nb_row, nb_box, tile_leaf, tile_begin,
                                                   kappa, shi, slo, y_near);
}

// ---------------------------------------------------------------------------------------------
// S2M: thread per direction k, leaf points streamed through shared memory.
// ---------------------------------------------------------------------------------------------
constexpr int S2M_TPB = 128;

__global__ void __launch_bounds__(S2M_TPB) s2m_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                      const double *__restrict__ cx,
                                                      const double *__restrict__ cy,
                                                      const double *__restrict__ cz, int32_t box0,
                                                      const double *__restrict__ ks, int64_t K,
                                                      double shi, double slo,
                                                      double2 *__restrict__ M) {
  __shared__ double2 tab[HFMM_TABLE];
  __shared__ double sx[S2M_TPB], sy[S2M_TPB], sz[S2M_TPB];
  __shared__ double2 sq[S2M_TPB];
  fill_exp_table(tab);
  const int32_t b = box0 + blockIdx.y;
  const int64_t k = (int64_t)blockIdx.x * S2M_TPB + threadIdx.x;
  const bool active = k < K;
  const double kx = active ? ks[k] : 0.0, ky = active ? ks[K + k] : 0.0, kz = active ? ks[2 * K + k] : 0.0;
  const double c0x = cx[b], c0y = cy[b], c0z = cz[b];
  const int64_t s0 = first[b], s1 = first[b + 1];
  double ar = 0.0, ai = 0.0;
  for (int64_t c0 = s0; c0 < s1; c0 += S2M_TPB) {
    const int cnt = (int)min((int64_t)S2M_TPB, s1 - c0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t j = c0 + threadIdx.x;
      sx[threadIdx.x] = pts.x[j] - c0x;
      sy[threadIdx.x] = pts.y[j] - c0y;
      sz[threadIdx.x] = pts.z[j] - c0z;
      sq[threadIdx.x] = pts.q[j];
    }
    __syncthreads();
#pragma unroll 4
    for (int u = 0; u < cnt; ++u) {
      const double ph = fma(kx, sx[u], fma(ky, sy[u], kz * sz[u]));
      const double2 e = cexpi_tab(ph, tab, shi, slo);
      const double2 q = sq[u];
      ar = fma(e.x, q.x, fma(-e.y, q.y, ar));
      ai = fma(e.x, q.y, fma(e.y, q.x, ai));
    }
  }
  if (active) M[(int64_t)b * K + k] = make_double2(ar, ai);
}

void launch_s2m(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, int32_t box0, int32_t box1, const double *ks, int64_t K,
                double2 *M, cudaStream_t s) {
  if (box1 <= box0) return;
  double shi, slo;
  step_split(&shi, &slo);
  dim3 grid((unsigned)((K + S2M_TPB - 1) / S2M_TPB), (unsigned)(box1 - box0));
  s2m_kernel<<<grid, S2M_TPB, 0, s>>>(pts, first, cx, cy, cz, box0, ks, K, shi, slo, M);
}

// ---------------------------------------------------------------------------------------------
// L2T: thread per target, directions streamed through shared memory.
// ---------------------------------------------------------------------------------------------
constexpr int L2T_TPB = 128;

__global__ void __launch_bounds__(L2T_TPB) l2t_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                      const double *__restrict__ cx,
                                                      const double *__restrict__ cy,
                                                      const double *__restrict__ cz,
                                                      const int32_t *__restrict__ tile_leaf,
                                                      const int64_t *__restrict__ tile_begin,
                                                      const double *__restrict__ ks, int64_t K,
                                                      const double2 *__restrict__ L, double w,
                                                      double shi, double slo,
                                                      double2 *__restrict__ y_far) {
  __shared__ double2 tab[HFMM_TABLE];
  __shared__ double skx[L2T_TPB], sky[L2T_TPB], skz[L2T_TPB];
  __shared__ double2 sl[L2T_TPB];
  fill_exp_table(tab);
  const int32_t leaf = tile_leaf[blockIdx.x];
  const int64_t i = tile_begin[blockIdx.x] + threadIdx.x;
  const bool active = i < first[leaf + 1];
  const double dx = active ? cx[leaf] - pts.x[i] : 0.0;   // c_a - x_i
  const double dy = active ? cy[leaf] - pts.y[i] : 0.0;
  const double dz = active ? cz[leaf] - pts.z[i] : 0.0;
  const double2 *Lb = L + (int64_t)leaf * K;
  double ar = 0.0, ai = 0.0;
  for (int64_t c0 = 0; c0 < K; c0 += L2T_TPB) {
    const int cnt = (int)min((int64_t)L2T_TPB, K - c0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t k = c0 + threadIdx.x;
      skx[threadIdx.x] = ks[k];
      sky[threadIdx.x] = ks[K + k];
      skz[threadIdx.x] = ks[2 * K + k];
      sl[threadIdx.x] = Lb[k];
    }
    __syncthreads();
#pragma unroll 4
    for (int u = 0; u < cnt; ++u) {
      const double ph = fma(skx[u], dx, fma(sky[u], dy, skz[u] * dz));
      const double2 e = cexpi_tab(ph, tab, shi, slo);
      const double2 l = sl[u];
      ar = fma(e.x, l.x, fma(-e.y, l.y, ar));
      ai = fma(e.x, l.y, fma(e.y, l.x, ai));
    }
  }
  if (active) y_far[i] = make_double2(w * ar, w * ai);
}

void launch_l2t(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, const int32_t *tile_leaf, const int64_t *tile_begin,
                int64_t ntiles, const double *ks, int64_t K, const double2 *L, double w,
                double2 *y_far, cudaStream_t s) {
  if (ntiles <= 0) return;
  double shi, slo;
  step_split(&shi, &slo);
  l2t_kernel<<<(unsigned)ntiles, L2T_TPB, 0, s>>>(pts, first, cx, cy, cz, tile_leaf, tile_begin, ks,
                                                   K, L, w, shi, slo, y_far);
}

// ---------------------------------------------------------------------------------------------
__global__ void permute_kernel(const double2 *__restrict__ q_in, const int64_t *__restrict__ perm,
                               double2 *__restrict__ q_sorted, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    q_sorted[i] = q_in[perm[i]];
}

void launch_permute_q(const double2 *q_in, const int64_t *perm, double2 *q_sorted, int64_t n,
                      cudaStream_t s) {
  if (n <= 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  permute_kernel<<<blocks, 256, 0, s>>>(q_in, perm, q_sorted, n);
}

__global__ void combine_kernel(const double2 *__restrict__ y_near, const double2 *__restrict__ y_far,
                               const int64_t *__restrict__ perm, double2 *__restrict__ y_out,
                               int64_t begin, int64_t end) {
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = y_near[i];
    if (y_far) {
      double2 b = y_far[i];
      a.x += b.x;
      a.y += b.y;
    }
    y_out[perm[i]] = a;
  }
}

void launch_combine(const double2 *y_near, const double2 *y_far, const int64_t *perm,
                    double2 *y_out, int64_t n, int64_t begin, int64_t end, cudaStream_t s) {
  (void)n;
  if (end <= begin) return;
  int blocks = (int)std::min<int64_t>((end - begin + 255) / 256, 148 * 16);
  combine_kernel<<<blocks, 256, 0, s>>>(y_near, y_far, perm, y_out, begin, end);
}

}  // namespace hfmm
