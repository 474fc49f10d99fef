// Point-wise FP64 kernels of the matvec (product code, sm_100a):
//   P2P  near field, eqn:FMM_FinalStep second term
//   S2M  initialisation M^L_a(s) = sum psi_i e^{i kappa s.(x_i - c_a)}
//   L2T  field computation int L e^{i kappa s.(c_a - x_i)} dS
//   permute / combine (Morton order <-> caller order)
// The three main kernels are bound by the FP64 pipe: one complex exponential per pair or per
// (point, direction).  Every phase arrives in units of the table step h = 2 pi/TAB (positions
// pre-scaled by kappa/h for P2P, directions kappa s/h for S2M/L2T, both at precompute), so e^{ix}
// (cexpi_u below) needs no range-reduction multiply: round to the nearest step with the
// 1.5 * 2^52 "magic number" (no FRND/F2I), exact remainder |r| <= 1/2 step, table
// e^{2 pi i k/TAB} in shared memory (TAB = 2048: 32 KB), Taylor polynomials of degree 3 (sin) and
// 4 (cos) whose truncation error (< 7e-17, |h r| <= pi/2048) is below the double rounding of the
// result: 12 FP64 instructions (TAB = 1024 needs a degree-5 sine, 13; A/B on C4: -1.6%).
// Each thread evaluates two items per source (ILP and source-load reuse).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "hfmm_impl.h"

namespace hfmm {

constexpr int TAB = TAB_STEPS;
constexpr double kMagic = 6755399441055744.0;          // 1.5 * 2^52
// Taylor coefficients in table-step units h = 2 pi / TAB:  sin(h r) = r (S1 + r^2 (S3 + r^2 S5)),
// cos(h r) = 1 + r^2 (C2 + r^2 C4), |r| <= 1/2 (|h r| <= pi/TAB, truncation (h r)^6/720).
constexpr double kH = 6.283185307179586476925286766559 / TAB;
constexpr double kS1 = kH, kS3 = -kH * kH * kH / 6.0, kS5 = kH * kH * kH * kH * kH / 120.0;
constexpr double kC2 = -kH * kH / 2.0, kC4 = kH * kH * kH * kH / 24.0;

// sin(h r) / (h-scaled) polynomial: degree 5 for TAB = 1024 (truncation 2e-18); degree 3 for
// TAB >= 2048 (|h r| <= pi/2048: truncation (h r)^5/120 <= 7e-17 < u = 2^-53).
__device__ __forceinline__ double sin_poly(double r, double r2) {
  if constexpr (TAB >= 2048) return r * fma(r2, kS3, kS1);
  else return r * fma(r2, fma(r2, kS5, kS3), kS1);
}

__device__ __forceinline__ void fill_exp_table(double2 *tab) {
  for (int t = threadIdx.x; t < TAB; t += blockDim.x) {
    double s, c;
    sincospi((double)t / (TAB / 2), &s, &c);
    tab[t] = make_double2(c, s);
  }
}

// e^{i h u} for a phase u given in table steps (h = 2 pi / TAB): u is rounded to the nearest
// integer k with the 1.5 * 2^52 magic number (exact for |u| < 2^51), the remainder r = u - k is
// exact (Sterbenz), and e^{i h u} = e^{2 pi i k / TAB} * e^{i h r}.
__device__ __forceinline__ double2 cexpi_u(double u, const double2 *__restrict__ tab) {
  const double t = u + kMagic;
  const int k = __double2loint(t);
  const double r = u - (t - kMagic);
  const double r2 = r * r;
  const double s = sin_poly(r, r2);
  const double c = fma(r2, fma(r2, kC4, kC2), 1.0);
  const double2 e = tab[k & (TAB - 1)];
  return make_double2(fma(e.x, c, -e.y * s), fma(e.x, s, e.y * c));
}

// e^{i h a b} for a phase given as a product a b (P2P: r^2 * (1/r)): the rounding to the nearest
// step comes straight from the exact product, k = round(a b) = fma(a, b, 1.5 * 2^52) - 1.5 * 2^52,
// and the remainder r = fma(a, b, -k) is rounded once -- one DMUL fewer than forming a b first.
#ifndef HFMM_P2P_I2F
#define HFMM_P2P_I2F 0   // A/B negative: C4 63.28 vs 62.99 ms (profiles/r02/mix_ab.txt)
#endif
__device__ __forceinline__ double2 cexpi_prod(double a, double b, const double2 *__restrict__ tab) {
  const double t = fma(a, b, kMagic);
  const int k = __double2loint(t);
#if HFMM_P2P_I2F   // A/B: k back to double on the conversion unit instead of a DADD on the FP64 pipe
  const double r = fma(a, b, -__int2double_rn(k));
#else
  const double r = fma(a, b, -(t - kMagic));
#endif
  const double r2 = r * r;
  const double s = sin_poly(r, r2);
  const double c = fma(r2, fma(r2, kC4, kC2), 1.0);
  const double2 e = tab[k & (TAB - 1)];
  return make_double2(fma(e.x, c, -e.y * s), fma(e.x, s, e.y * c));
}

// 1/sqrt(r2) for r2 > 0: hardware approximation of the high word, one cubic Newton step.
// HFMM_P2P_RSQ32 (A/B): seed from the FP32 MUFU.RSQ of the rounded r2 instead of MUFU.RSQ64H --
// slower (C4 70.2 vs 68.2 ms: the two F2F conversions cost more than the 64-bit MUFU seed;
// profiles/r02/p2p_rsq32_ab.txt).
#ifndef HFMM_P2P_RSQ32
#define HFMM_P2P_RSQ32 0
#endif
#ifndef HFMM_RSQ_FORM
#define HFMM_RSQ_FORM 1
#endif
#ifndef HFMM_P2P_UNROLL
#define HFMM_P2P_UNROLL 4   // 4 vs 2: C4 62.86 vs 62.99 ms, C5 719.7 vs 722.8 (profiles/r02/mix_ab.txt)
#endif
__device__ __forceinline__ double rsqrt_fast(double r2) {
  double y;
#if HFMM_P2P_RSQ32
  y = (double)rsqrtf(__double2float_rn(r2));
#else
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
#endif
  const double e = fma(-r2, y * y, 1.0);
#if HFMM_RSQ_FORM == 0
  return fma(y * e, fma(e, 0.375, 0.5), y);
#else
  return y * fma(e, fma(e, 0.375, 0.5), 1.0);   // every DFMA reads <= 2 vector registers
#endif
}

// ---------------------------------------------------------------------------------------------
// P2P.  Positions are stored pre-scaled to table steps, u = x * S with
// S = kappa TAB / (2 pi), so that kappa R = h |u_i - u_j| and
//     G = e^{i kappa R} / R = S * e^{i h R_u} / R_u,      R_u = |u_i - u_j|;
// the kernels accumulate e^{i h R_u} / R_u and multiply by S once per target (per item).
// Work items are (t0, t1, s0, s1): targets [t0, t1) (<= 256, 2 per thread), sources [s0, s1)
// streamed through shared memory in chunks of 128.
//   ordered   rows only; DIAG masks the self pair (R = 0 <=> i = j: coincident distinct
//             points are rejected at build_tree) when the source range contains the targets
//   symmetric disjoint ranges: each unordered pair evaluated once, G q_j added to y_i (rows, in
//             registers) and G q_i to y_j (columns: systolic warp reduction, below)
// ---------------------------------------------------------------------------------------------
constexpr int P2P_TPB = P2P_THREADS;
constexpr int kP2PUnroll = HFMM_P2P_UNROLL;   // source steps unrolled in the full-tile symmetric loop (A/B)
// PT = targets per thread (tile = PT * P2P_TPB), MINB = resident CTAs per SM asked of ptxas;
// instantiated as (8, 1), (4, HFMM_P2P_MINB) and (3, 4) -- the plan picks one per matvec (hfmm.cu)

__device__ __forceinline__ double2 green_u(double tx, double ty, double tz, double xs, double ys, double zs,
                                           const double2 *tab) {
  const double dx = tx - xs, dy = ty - ys, dz = tz - zs;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ri = rsqrt_fast(r2);
  const double2 e = cexpi_prod(r2, ri, tab);  // e^{i h R_u}, R_u = r2 / sqrt(r2)
  return make_double2(e.x * ri, e.y * ri);
}

// Outputs: y_near += (atomics, default), or -- deterministic mode (part != nullptr) -- the item's
// row / column partial sums written to part[slot[2 item] + row], part[slot[2 item + 1] + column],
// summed per point in a fixed order afterwards (p2p_reduce_kernel): bitwise reproducible.
template <bool DIAG, int PT, int MINB>
__global__ void __launch_bounds__(P2P_TPB, MINB) p2p_ord_kernel(PointsU pts,
                                                                        const int64_t *__restrict__ items,
                                                                        double scale, double2 *__restrict__ y_near,
                                                                        double2 *__restrict__ part,
                                                                        const int64_t *__restrict__ slot) {
  __shared__ double2 tab[TAB];
  __shared__ double sx[P2P_TPB], sy[P2P_TPB], sz[P2P_TPB];
  __shared__ double2 sq[P2P_TPB];
  fill_exp_table(tab);
  const int64_t *it = items + 4 * (int64_t)blockIdx.x;
  const int64_t t1 = it[1], s0 = it[2], s1 = it[3];
  double tx[PT], ty[PT], tz[PT], ar[PT], ai[PT];
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int64_t i = it[0] + threadIdx.x + p * P2P_TPB;
    // inactive lanes evaluate far-away dummy targets (results discarded)
    tx[p] = i < t1 ? pts.ux[i] : 1e30, ty[p] = i < t1 ? pts.uy[i] : 0.0, tz[p] = i < t1 ? pts.uz[i] : 0.0;
    ar[p] = ai[p] = 0.0;
  }
  for (int64_t c0 = s0; c0 < s1; c0 += P2P_TPB) {
    const int cnt = (int)min((int64_t)P2P_TPB, s1 - c0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t j = c0 + threadIdx.x;
      sx[threadIdx.x] = pts.ux[j];
      sy[threadIdx.x] = pts.uy[j];
      sz[threadIdx.x] = pts.uz[j];
      sq[threadIdx.x] = pts.q[j];
    }
    __syncthreads();
#pragma unroll 2
    for (int u = 0; u < cnt; ++u) {
      const double xs = sx[u], ys = sy[u], zs = sz[u];
      const double2 q = sq[u];
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const double dx = tx[p] - xs, dy = ty[p] - ys, dz = tz[p] - zs;
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        double ri = rsqrt_fast(r2);
        if (DIAG) ri = (r2 > 0.0) ? ri : 0.0;  // self pair excluded
        const double2 e = cexpi_prod(r2, ri, tab);
        const double gr = e.x * ri, gi = e.y * ri;
        ar[p] = fma(gr, q.x, fma(-gi, q.y, ar[p]));
        ai[p] = fma(gr, q.y, fma(gi, q.x, ai[p]));
      }
    }
  }
  // y_near is zeroed before the P2P launches; every item adds into its target rows
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int64_t i = it[0] + threadIdx.x + p * P2P_TPB;
    if (i >= t1) continue;
    if (part) part[slot[2 * (int64_t)blockIdx.x] + (i - it[0])] = make_double2(scale * ar[p], scale * ai[p]);
    else atomicAdd(&y_near[i].x, scale * ar[p]), atomicAdd(&y_near[i].y, scale * ai[p]);
  }
}

// Symmetric item: column sums use a systolic warp reduction -- in a block of 32 sources, lane t
// processes source (t + u) mod 32 at step u and passes the running column accumulator to lane
// t - 1, so after 32 steps lane t holds the warp sum of source t (2 shuffles per step instead of
// a 5-level butterfly per source); the 4 warps combine in shared memory, one atomic per source.
// Each source loaded from shared memory serves PT targets of the lane.
// DS (diagonal tile, targets == sources, <= PT x P2P_TPB points): each unordered pair once -- 32-point
// block pairs (target block tb = warp + (P2P_TPB / 32) p, source block sb) with tb < sb in full, tb == sb for half
// of the systolic rotation (steps 1..15 and lanes < 16 of step 16; step 0 is the excluded self pair,
// P:90), tb > sb skipped (warp-uniform branches).
// One 32-source block of the symmetric item for a warp whose first NP target rows p (targets
// t0 + 32 warp + 128 p + lane) hold live targets: rows p >= NP lie wholly past the tile's end
// and are not evaluated at all (warp-row granularity instead of the tile's; the dispatch below is
// warp-uniform and outside the source loop, so each variant keeps the straight-line schedule).
template <bool DS, int PT, int NP>
__device__ __forceinline__ void p2p_sym_block(const double (&tx)[PT], const double (&ty)[PT], const double (&tz)[PT],
                                              const double2 (&tq)[PT], double (&ar)[PT], double (&ai)[PT],
                                              const double *sx, const double *sy, const double *sz,
                                              const double2 *sq, const double2 *tab, int lane, int warp,
                                              int base, int sb, double &cr_out, double &ci_out) {
  double cr = 0.0, ci = 0.0;
#pragma unroll 2   // (4x here: C5 at eps/10, row skipping, 205.7 vs 200.3 ms)
  for (int u = 0; u < 32; ++u) {
    const int s = base + ((lane + u) & 31);
    const double xs = sx[s], ys = sy[s], zs = sz[s];
    const double2 qs = sq[s];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double w = 1.0;
      if (DS) {
        const int tb = warp + (P2P_TPB / 32) * p;
        if (tb > sb) continue;
        if (tb == sb) {
          if (u == 0 || u > 16) continue;
          if (u == 16 && lane >= 16) w = 0.0;   // the other half of the antipodal step
        }
      }
      double2 g = green_u(tx[p], ty[p], tz[p], xs, ys, zs, tab);
      if (DS) g = make_double2(g.x * w, g.y * w);
      ar[p] = fma(g.x, qs.x, fma(-g.y, qs.y, ar[p]));
      ai[p] = fma(g.x, qs.y, fma(g.y, qs.x, ai[p]));
      cr = fma(g.x, tq[p].x, fma(-g.y, tq[p].y, cr));
      ci = fma(g.x, tq[p].y, fma(g.y, tq[p].x, ci));
    }
    cr = __shfl_sync(0xffffffffu, cr, (lane + 1) & 31);   // accumulator follows its source
    ci = __shfl_sync(0xffffffffu, ci, (lane + 1) & 31);
  }
  cr_out = cr, ci_out = ci;
}

template <bool DS, int PT, int NP>
__device__ __forceinline__ void p2p_sym_dispatch(int np, const double (&tx)[PT], const double (&ty)[PT],
                                                 const double (&tz)[PT], const double2 (&tq)[PT], double (&ar)[PT],
                                                 double (&ai)[PT], const double *sx, const double *sy,
                                                 const double *sz, const double2 *sq, const double2 *tab, int lane,
                                                 int warp, int base, int sb, double &cr, double &ci) {
  if constexpr (NP == 0) {
    cr = ci = 0.0;   // no live target in this warp: its column partial sums are zero
  } else {
    if (np >= NP) p2p_sym_block<DS, PT, NP>(tx, ty, tz, tq, ar, ai, sx, sy, sz, sq, tab, lane, warp, base, sb, cr, ci);
    else p2p_sym_dispatch<DS, PT, NP - 1>(np, tx, ty, tz, tq, ar, ai, sx, sy, sz, sq, tab, lane, warp, base, sb, cr, ci);
  }
}

template <bool DS, int PT, int MINB, bool RS>
__global__ void __launch_bounds__(P2P_TPB, MINB) p2p_sym_kernel(PointsU pts,
                                                                        const int64_t *__restrict__ items,
                                                                        double scale, double3 dummy_t,
                                                                        double3 dummy_s,
                                                                        double2 *__restrict__ y_near,
                                                                        double2 *__restrict__ part,
                                                                        const int64_t *__restrict__ slot) {
  __shared__ double2 tab[TAB];
  __shared__ double sx[P2P_TPB], sy[P2P_TPB], sz[P2P_TPB];
  __shared__ double2 sq[P2P_TPB];
  __shared__ double2 col[P2P_TPB / 32][P2P_TPB];
  fill_exp_table(tab);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t *it = items + 4 * (int64_t)blockIdx.x;
  const int64_t t1 = it[1], s0 = it[2], s1 = it[3];
  double tx[PT], ty[PT], tz[PT], ar[PT], ai[PT];
  double2 tq[PT];
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int64_t i = it[0] + threadIdx.x + p * P2P_TPB;
    const bool v = i < t1;
    // inactive targets: far dummy position, zero charge (their column contributions vanish)
    tx[p] = v ? pts.ux[i] : dummy_t.x, ty[p] = v ? pts.uy[i] : dummy_t.y, tz[p] = v ? pts.uz[i] : dummy_t.z;
    tq[p] = v ? pts.q[i] : make_double2(0.0, 0.0);
    ar[p] = ai[p] = 0.0;
  }
  // live target rows of this warp: row p holds targets t0 + 32 warp + 128 p + lane
  int np_w = PT;
  if (RS) {
    const int64_t left = t1 - (it[0] + 32 * warp);
    np_w = left <= 0 ? 0 : (int)min((int64_t)PT, (left + P2P_TPB - 1) / P2P_TPB);
  }
  for (int64_t c0 = s0; c0 < s1; c0 += P2P_TPB) {
    const int cnt = (int)min((int64_t)P2P_TPB, s1 - c0);
    __syncthreads();
    {
      const int t = threadIdx.x;
      const bool v = t < cnt;
      const int64_t j = c0 + t;
      sx[t] = v ? pts.ux[j] : dummy_s.x;   // padded sources: far dummy, zero charge
      sy[t] = v ? pts.uy[j] : dummy_s.y;
      sz[t] = v ? pts.uz[j] : dummy_s.z;
      sq[t] = v ? pts.q[j] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int nblk = (cnt + 31) >> 5;
    for (int blk = 0; blk < nblk; ++blk) {
      const int base = blk << 5;
      const int sb = (int)((c0 - s0) >> 5) + blk;  // source block (DS)
      double cr = 0.0, ci = 0.0;
      if (RS) {   // every tile through the per-row-count variants (full tiles through the inline
                  // loop below instead: C4 68.1 vs 67.1 ms with skipping on, profiles/r02/rowskip_ab2.txt)
        p2p_sym_dispatch<DS, PT, PT>(np_w, tx, ty, tz, tq, ar, ai, sx, sy, sz, sq, tab, lane, warp, base, sb, cr, ci);
      } else {  // all PT rows (the full-tile loop, inline)
#pragma unroll kP2PUnroll
        for (int u = 0; u < 32; ++u) {
          const int s = base + ((lane + u) & 31);
          const double xs = sx[s], ys = sy[s], zs = sz[s];
          const double2 qs = sq[s];
#pragma unroll
          for (int p = 0; p < PT; ++p) {
            double w = 1.0;
            if (DS) {
              const int tb = warp + (P2P_TPB / 32) * p;
              if (tb > sb) continue;
              if (tb == sb) {
                if (u == 0 || u > 16) continue;
                if (u == 16 && lane >= 16) w = 0.0;   // the other half of the antipodal step
              }
            }
            double2 g = green_u(tx[p], ty[p], tz[p], xs, ys, zs, tab);
            if (DS) g = make_double2(g.x * w, g.y * w);
            ar[p] = fma(g.x, qs.x, fma(-g.y, qs.y, ar[p]));
            ai[p] = fma(g.x, qs.y, fma(g.y, qs.x, ai[p]));
            cr = fma(g.x, tq[p].x, fma(-g.y, tq[p].y, cr));
            ci = fma(g.x, tq[p].y, fma(g.y, tq[p].x, ci));
          }
          cr = __shfl_sync(0xffffffffu, cr, (lane + 1) & 31);   // accumulator follows its source
          ci = __shfl_sync(0xffffffffu, ci, (lane + 1) & 31);
        }
      }
      col[warp][base + lane] = make_double2(cr, ci);
    }
    __syncthreads();
    if (threadIdx.x < cnt) {
      double2 sum = col[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < P2P_TPB / 32; ++w) sum.x += col[w][threadIdx.x].x, sum.y += col[w][threadIdx.x].y;
      if (part) {
        part[slot[2 * (int64_t)blockIdx.x + 1] + (c0 - s0) + threadIdx.x] = make_double2(scale * sum.x, scale * sum.y);
      } else {
        atomicAdd(&y_near[c0 + threadIdx.x].x, scale * sum.x);
        atomicAdd(&y_near[c0 + threadIdx.x].y, scale * sum.y);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    const int64_t i = it[0] + threadIdx.x + p * P2P_TPB;
    if (i >= t1) continue;
    if (part) part[slot[2 * (int64_t)blockIdx.x] + (i - it[0])] = make_double2(scale * ar[p], scale * ai[p]);
    else atomicAdd(&y_near[i].x, scale * ar[p]), atomicAdd(&y_near[i].y, scale * ai[p]);
  }
}

// Deterministic mode: y_near[i] = sum over the partials of point i in the order of its list.
__global__ void p2p_reduce_kernel(const double2 *__restrict__ part, const int64_t *__restrict__ row_ptr,
                                  const int64_t *__restrict__ idx, int64_t n, double2 *__restrict__ y_near) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      const double2 v = part[idx[e]];
      acc.x += v.x, acc.y += v.y;
    }
    y_near[i] = acc;
  }
}

void launch_p2p_reduce(const double2 *part, const int64_t *row_ptr, const int64_t *idx, int64_t n, double2 *y_near,
                       cudaStream_t s) {
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  p2p_reduce_kernel<<<blocks, 256, 0, s>>>(part, row_ptr, idx, n, y_near);
}

template <int PT, int MINB, bool RS>
static void launch_p2p_items_t(PointsU pts, const int64_t *items, int64_t nitems, int kind, double scale,
                               const double dummy_t[3], const double dummy_s[3], double2 *y_near, double2 *part,
                               const int64_t *slot, cudaStream_t s) {
  if (kind == P2P_SYM || kind == P2P_DSYM) {
    auto kern = kind == P2P_SYM ? p2p_sym_kernel<false, PT, MINB, RS> : p2p_sym_kernel<true, PT, MINB, RS>;
    kern<<<(unsigned)nitems, P2P_TPB, 0, s>>>(pts, items, scale, make_double3(dummy_t[0], dummy_t[1], dummy_t[2]),
                                             make_double3(dummy_s[0], dummy_s[1], dummy_s[2]), y_near, part, slot);
  }
  else if (kind == P2P_DIAG)
    p2p_ord_kernel<true, PT, MINB><<<(unsigned)nitems, P2P_TPB, 0, s>>>(pts, items, scale, y_near, part, slot);
  else
    p2p_ord_kernel<false, PT, MINB><<<(unsigned)nitems, P2P_TPB, 0, s>>>(pts, items, scale, y_near, part, slot);
}

void launch_p2p_items(PointsU pts, const int64_t *items, int64_t nitems, int kind, double scale,
                      const double dummy_t[3], const double dummy_s[3], double2 *y_near, cudaStream_t s, int pt,
                      double2 *part, const int64_t *slot, bool rowskip) {
  if (nitems <= 0) return;
  if (pt == 3 && rowskip)
    launch_p2p_items_t<3, 4, true>(pts, items, nitems, kind, scale, dummy_t, dummy_s, y_near, part, slot, s);
  else if (pt == 3)
    launch_p2p_items_t<3, 4, false>(pts, items, nitems, kind, scale, dummy_t, dummy_s, y_near, part, slot, s);
  else if (pt == 8)
    launch_p2p_items_t<8, 1, false>(pts, items, nitems, kind, scale, dummy_t, dummy_s, y_near, part, slot, s);
  else if (rowskip)
    launch_p2p_items_t<4, HFMM_P2P_MINB, true>(pts, items, nitems, kind, scale, dummy_t, dummy_s, y_near, part, slot, s);
  else
    launch_p2p_items_t<4, HFMM_P2P_MINB, false>(pts, items, nitems, kind, scale, dummy_t, dummy_s, y_near, part, slot, s);
}

// ---------------------------------------------------------------------------------------------
// S2M: two directions per thread (k, k + 128), leaf points streamed through shared memory.
// ---------------------------------------------------------------------------------------------
constexpr int S2M_TPB = 128;

__global__ void __launch_bounds__(S2M_TPB, 5) s2m_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                         const double *__restrict__ cx,
                                                         const double *__restrict__ cy,
                                                         const double *__restrict__ cz, int32_t box0,
                                                         const double *__restrict__ ks, int64_t K,
                                                         double2 *__restrict__ M) {
  __shared__ double2 tab[TAB];
  __shared__ double sx[S2M_TPB], sy[S2M_TPB], sz[S2M_TPB];
  __shared__ double2 sq[S2M_TPB];
  fill_exp_table(tab);
  const int32_t b = box0 + blockIdx.x;   // boxes on x (gridDim.y is limited to 65535)
  const int64_t k0 = (int64_t)blockIdx.y * (2 * S2M_TPB) + threadIdx.x, k1 = k0 + S2M_TPB;
  const double kx0 = k0 < K ? ks[k0] : 0.0, ky0 = k0 < K ? ks[K + k0] : 0.0, kz0 = k0 < K ? ks[2 * K + k0] : 0.0;
  const double kx1 = k1 < K ? ks[k1] : 0.0, ky1 = k1 < K ? ks[K + k1] : 0.0, kz1 = k1 < K ? ks[2 * K + k1] : 0.0;
  const double c0x = cx[b], c0y = cy[b], c0z = cz[b];
  const int64_t s0 = first[b], s1 = first[b + 1];
  double a0r = 0.0, a0i = 0.0, a1r = 0.0, a1i = 0.0;
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
#pragma unroll 2
    for (int u = 0; u < cnt; ++u) {
      const double dx = sx[u], dy = sy[u], dz = sz[u];
      const double2 q = sq[u];
      const double2 e0 = cexpi_u(fma(kx0, dx, fma(ky0, dy, kz0 * dz)), tab);
      a0r = fma(e0.x, q.x, fma(-e0.y, q.y, a0r));
      a0i = fma(e0.x, q.y, fma(e0.y, q.x, a0i));
      const double2 e1 = cexpi_u(fma(kx1, dx, fma(ky1, dy, kz1 * dz)), tab);
      a1r = fma(e1.x, q.x, fma(-e1.y, q.y, a1r));
      a1i = fma(e1.x, q.y, fma(e1.y, q.x, a1i));
    }
  }
  if (k0 < K) M[(int64_t)b * K + k0] = make_double2(a0r, a0i);
  if (k1 < K) M[(int64_t)b * K + k1] = make_double2(a1r, a1i);
}

void launch_s2m(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, int32_t box0, int32_t box1, const double *ks, int64_t K,
                double2 *M, cudaStream_t s) {
  if (box1 <= box0) return;
  dim3 grid((unsigned)(box1 - box0), (unsigned)((K + 2 * S2M_TPB - 1) / (2 * S2M_TPB)));
  s2m_kernel<<<grid, S2M_TPB, 0, s>>>(pts, first, cx, cy, cz, box0, ks, K, M);
}

// ---------------------------------------------------------------------------------------------
// L2T: two targets per thread (tile of 256 targets), directions streamed through shared memory.
// ---------------------------------------------------------------------------------------------
constexpr int L2T_TPB = 128;

__global__ void __launch_bounds__(L2T_TPB, 5) l2t_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                         const double *__restrict__ cx,
                                                         const double *__restrict__ cy,
                                                         const double *__restrict__ cz,
                                                         const int32_t *__restrict__ tile_leaf,
                                                         const int64_t *__restrict__ tile_begin,
                                                         const double *__restrict__ ks, int64_t K,
                                                         const double2 *__restrict__ L, double w,
                                                         const double *__restrict__ wk,
                                                         double2 *__restrict__ y_far) {
  __shared__ double2 tab[TAB];
  __shared__ double skx[L2T_TPB], sky[L2T_TPB], skz[L2T_TPB];
  __shared__ double2 sl[L2T_TPB];
  fill_exp_table(tab);
  const int32_t leaf = tile_leaf[blockIdx.x];
  const int64_t tend = first[leaf + 1];
  const int64_t i0 = tile_begin[blockIdx.x] + threadIdx.x, i1 = i0 + L2T_TPB;
  const double ccx = cx[leaf], ccy = cy[leaf], ccz = cz[leaf];
  const double dx0 = i0 < tend ? ccx - pts.x[i0] : 0.0, dy0 = i0 < tend ? ccy - pts.y[i0] : 0.0,
               dz0 = i0 < tend ? ccz - pts.z[i0] : 0.0;   // c_a - x_i
  const double dx1 = i1 < tend ? ccx - pts.x[i1] : 0.0, dy1 = i1 < tend ? ccy - pts.y[i1] : 0.0,
               dz1 = i1 < tend ? ccz - pts.z[i1] : 0.0;
  const double2 *Lb = L + (int64_t)leaf * K;
  double a0r = 0.0, a0i = 0.0, a1r = 0.0, a1i = 0.0;
  for (int64_t c0 = 0; c0 < K; c0 += L2T_TPB) {
    const int cnt = (int)min((int64_t)L2T_TPB, K - c0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t k = c0 + threadIdx.x;
      skx[threadIdx.x] = ks[k];
      sky[threadIdx.x] = ks[K + k];
      skz[threadIdx.x] = ks[2 * K + k];
      const double2 lv = Lb[k];
      const double wt = wk ? wk[k] : 1.0;  // per-point quadrature weight (ragged rows, R-15)
      sl[threadIdx.x] = make_double2(wt * lv.x, wt * lv.y);
    }
    __syncthreads();
#pragma unroll 2
    for (int u = 0; u < cnt; ++u) {
      const double kx = skx[u], ky = sky[u], kz = skz[u];
      const double2 l = sl[u];
      const double2 e0 = cexpi_u(fma(kx, dx0, fma(ky, dy0, kz * dz0)), tab);
      a0r = fma(e0.x, l.x, fma(-e0.y, l.y, a0r));
      a0i = fma(e0.x, l.y, fma(e0.y, l.x, a0i));
      const double2 e1 = cexpi_u(fma(kx, dx1, fma(ky, dy1, kz * dz1)), tab);
      a1r = fma(e1.x, l.x, fma(-e1.y, l.y, a1r));
      a1i = fma(e1.x, l.y, fma(e1.y, l.x, a1i));
    }
  }
  if (wk) w = 1.0;
  if (i0 < tend) y_far[i0] = make_double2(w * a0r, w * a0i);
  if (i1 < tend) y_far[i1] = make_double2(w * a1r, w * a1i);
}

void launch_l2t(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, const int32_t *tile_leaf, const int64_t *tile_begin,
                int64_t ntiles, const double *ks, int64_t K, const double2 *L, double w,
                const double *wk, double2 *y_far, cudaStream_t s) {
  if (ntiles <= 0) return;
  l2t_kernel<<<(unsigned)ntiles, L2T_TPB, 0, s>>>(pts, first, cx, cy, cz, tile_leaf, tile_begin, ks, K, L, w, wk,
                                                   y_far);
}

// ---------------------------------------------------------------------------------------------
// Small-box S2M / L2T (source level D_s below L_f, R-14: a few to a few tens of points
// per box, K of a few hundred).  Persistent CTAs (the e^{ih k} table is filled once per CTA),
// one warp per box.
//   S2M: lanes over directions (k0 + lane, k0 + 32 + lane), the box's points staged 32 at a
//        time in a per-warp shared buffer (positions relative to the centre) and broadcast.
//   L2T: lane = (point p = lane % P, slice = lane / P) with P = the next power of two >= the
//        box's points (<= 32) and 32/P slices of the directions; slices reduced by shuffles.
// ---------------------------------------------------------------------------------------------
constexpr int SMALL_TPB = 128;
#ifndef HFMM_L2T_V2
#define HFMM_L2T_V2 1  // L2T with directions on lanes (0: point-on-lane kernel, A/B)
#endif
constexpr int SMALL_WARPS = SMALL_TPB / 32;

__global__ void __launch_bounds__(SMALL_TPB) s2m_warp_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                             const double *__restrict__ cx,
                                                             const double *__restrict__ cy,
                                                             const double *__restrict__ cz, int32_t box0,
                                                             int32_t box1, const double *__restrict__ ks,
                                                             int64_t K, double2 *__restrict__ M) {
  __shared__ double2 tab[TAB];
  __shared__ double wx[SMALL_WARPS][32], wy[SMALL_WARPS][32], wz[SMALL_WARPS][32];
  __shared__ double2 wq[SMALL_WARPS][32];
  fill_exp_table(tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * SMALL_WARPS;
  for (int64_t b = box0 + (int64_t)blockIdx.x * SMALL_WARPS + warp; b < box1; b += nwarps) {
    const int64_t s0 = first[b], s1 = first[b + 1];
    const double c0x = cx[b], c0y = cy[b], c0z = cz[b];
    const bool one_chunk = s1 - s0 <= 32;
    for (int64_t k0 = 0; k0 < K; k0 += 64) {
      const int64_t ka = k0 + lane, kb = ka + 32;
      const double kxa = ka < K ? ks[ka] : 0.0, kya = ka < K ? ks[K + ka] : 0.0, kza = ka < K ? ks[2 * K + ka] : 0.0;
      const double kxb = kb < K ? ks[kb] : 0.0, kyb = kb < K ? ks[K + kb] : 0.0, kzb = kb < K ? ks[2 * K + kb] : 0.0;
      double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
      for (int64_t j0 = s0; j0 < s1; j0 += 32) {
        const int cnt = (int)min((int64_t)32, s1 - j0);
        if (!one_chunk || k0 == 0) {
          __syncwarp();
          if (lane < cnt) {
            const int64_t j = j0 + lane;
            wx[warp][lane] = pts.x[j] - c0x;
            wy[warp][lane] = pts.y[j] - c0y;
            wz[warp][lane] = pts.z[j] - c0z;
            wq[warp][lane] = pts.q[j];
          }
          __syncwarp();
        }
#pragma unroll 2
        for (int u = 0; u < cnt; ++u) {
          const double dx = wx[warp][u], dy = wy[warp][u], dz = wz[warp][u];
          const double2 q = wq[warp][u];
          const double2 ea = cexpi_u(fma(kxa, dx, fma(kya, dy, kza * dz)), tab);
          ar = fma(ea.x, q.x, fma(-ea.y, q.y, ar));
          ai = fma(ea.x, q.y, fma(ea.y, q.x, ai));
          const double2 eb = cexpi_u(fma(kxb, dx, fma(kyb, dy, kzb * dz)), tab);
          br = fma(eb.x, q.x, fma(-eb.y, q.y, br));
          bi = fma(eb.x, q.y, fma(eb.y, q.x, bi));
        }
      }
      if (ka < K) M[b * K + ka] = make_double2(ar, ai);
      if (kb < K) M[b * K + kb] = make_double2(br, bi);
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(SMALL_TPB) l2t_warp_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                             const double *__restrict__ cx,
                                                             const double *__restrict__ cy,
                                                             const double *__restrict__ cz, int32_t box0,
                                                             int32_t box1, const double *__restrict__ ks,
                                                             int64_t K, const double2 *__restrict__ L, double w,
                                                             const double *__restrict__ wk,
                                                             double2 *__restrict__ y_far) {
  __shared__ double2 tab[TAB];
  fill_exp_table(tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * SMALL_WARPS;
  for (int64_t b = box0 + (int64_t)blockIdx.x * SMALL_WARPS + warp; b < box1; b += nwarps) {
    const int64_t s0 = first[b], s1 = first[b + 1];
    const int64_t nb = s1 - s0;
    int P = 1;
    while (P < nb && P < 32) P <<= 1;
    const int S = 32 / P, slice = lane / P;
    const double ccx = cx[b], ccy = cy[b], ccz = cz[b];
    const double2 *Lb = L + b * K;
    for (int64_t p0 = s0; p0 < s1; p0 += P) {
      const int64_t i = p0 + (lane & (P - 1));
      const bool valid = i < s1;
      const double dx = valid ? ccx - pts.x[i] : 0.0, dy = valid ? ccy - pts.y[i] : 0.0,
                   dz = valid ? ccz - pts.z[i] : 0.0;   // c_a - x_i
      double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
      for (int64_t k = slice; k < K; k += 2 * S) {
        {
          double2 l = Lb[k];
          if (wk) l = make_double2(wk[k] * l.x, wk[k] * l.y);  // per-point weight (ragged rows, R-15)
          const double2 e = cexpi_u(fma(ks[k], dx, fma(ks[K + k], dy, ks[2 * K + k] * dz)), tab);
          ar = fma(e.x, l.x, fma(-e.y, l.y, ar));
          ai = fma(e.x, l.y, fma(e.y, l.x, ai));
        }
        const int64_t k2 = k + S;
        if (k2 < K) {
          double2 l = Lb[k2];
          if (wk) l = make_double2(wk[k2] * l.x, wk[k2] * l.y);
          const double2 e = cexpi_u(fma(ks[k2], dx, fma(ks[K + k2], dy, ks[2 * K + k2] * dz)), tab);
          br = fma(e.x, l.x, fma(-e.y, l.y, br));
          bi = fma(e.x, l.y, fma(e.y, l.x, bi));
        }
      }
      ar += br, ai += bi;
      for (int off = P; off < 32; off <<= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, off);
        ai += __shfl_xor_sync(0xffffffffu, ai, off);
      }
      const double ws = wk ? 1.0 : w;
      if (slice == 0 && valid) y_far[i] = make_double2(ws * ar, ws * ai);
    }
  }
}

// L2T, directions on lanes (the S2M layout): lane holds directions (k0 + lane, k0 + 32 + lane)
// with their L values and kappa s in registers, the box's points are broadcast from shared memory
// 32 at a time, and each point's partial sum is reduced across the warp (5 xor-shuffle levels);
// lane p keeps the running sum of point p of the current 32-point batch.  Two evaluations per
// lane per point with no global load in the inner loop.
__global__ void __launch_bounds__(SMALL_TPB) l2t_warp2_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                              const double *__restrict__ cx,
                                                              const double *__restrict__ cy,
                                                              const double *__restrict__ cz, int32_t box0,
                                                              int32_t box1, const double *__restrict__ ks,
                                                              int64_t K, const double2 *__restrict__ L, double w,
                                                              const double *__restrict__ wk,
                                                              double2 *__restrict__ y_far) {
  __shared__ double2 tab[TAB];
  __shared__ double wx[SMALL_WARPS][32], wy[SMALL_WARPS][32], wz[SMALL_WARPS][32];
  fill_exp_table(tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * SMALL_WARPS;
  const double ws = wk ? 1.0 : w;
  for (int64_t b = box0 + (int64_t)blockIdx.x * SMALL_WARPS + warp; b < box1; b += nwarps) {
    const int64_t s0 = first[b], s1 = first[b + 1];
    const double c0x = cx[b], c0y = cy[b], c0z = cz[b];
    const double2 *Lb = L + b * K;
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {  // batches of 32 points
      const int cnt = (int)min((int64_t)32, s1 - j0);
      __syncwarp();
      if (lane < cnt) {  // c_a - x_i
        wx[warp][lane] = c0x - pts.x[j0 + lane];
        wy[warp][lane] = c0y - pts.y[j0 + lane];
        wz[warp][lane] = c0z - pts.z[j0 + lane];
      }
      __syncwarp();
      double yr = 0.0, yi = 0.0;  // lane p: point j0 + p
      for (int64_t k0 = 0; k0 < K; k0 += 64) {
        const int64_t ka = k0 + lane, kb = ka + 32;
        const bool va = ka < K, vb = kb < K;
        const double kxa = va ? ks[ka] : 0.0, kya = va ? ks[K + ka] : 0.0, kza = va ? ks[2 * K + ka] : 0.0;
        const double kxb = vb ? ks[kb] : 0.0, kyb = vb ? ks[K + kb] : 0.0, kzb = vb ? ks[2 * K + kb] : 0.0;
        double2 la = va ? Lb[ka] : make_double2(0.0, 0.0), lb = vb ? Lb[kb] : make_double2(0.0, 0.0);
        if (wk) {  // per-point weights (ragged rows, R-15)
          const double wa = va ? wk[ka] : 0.0, wb = vb ? wk[kb] : 0.0;
          la = make_double2(wa * la.x, wa * la.y), lb = make_double2(wb * lb.x, wb * lb.y);
        }
        for (int p = 0; p < cnt; ++p) {
          const double dx = wx[warp][p], dy = wy[warp][p], dz = wz[warp][p];
          const double2 ea = cexpi_u(fma(kxa, dx, fma(kya, dy, kza * dz)), tab);
          const double2 eb = cexpi_u(fma(kxb, dx, fma(kyb, dy, kzb * dz)), tab);
          double pr = fma(ea.x, la.x, fma(-ea.y, la.y, fma(eb.x, lb.x, -eb.y * lb.y)));
          double pi = fma(ea.x, la.y, fma(ea.y, la.x, fma(eb.x, lb.y, eb.y * lb.x)));
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            pr += __shfl_xor_sync(0xffffffffu, pr, off);
            pi += __shfl_xor_sync(0xffffffffu, pi, off);
          }
          if (lane == p) yr += pr, yi += pi;
        }
      }
      if (lane < cnt) y_far[j0 + lane] = make_double2(ws * yr, ws * yi);
    }
  }
}

// L2T v3: directions on lanes like v2, but each lane accumulates its directions' terms for a
// sub-batch of PB points over the whole direction loop and the warp reduces each point ONCE
// (v2 reduced every point after every 64 directions: 20 SHFL + 10 DADD per point and chunk, about
// as much shuffle-pipe time as the 48 FP64 instructions of the chunk).  Per (point, 32 directions):
// phase 3 + e^{ix} 12 + MAC 4 FP64 instructions per lane; the 5-level butterfly per point is
// amortised over K / 32 chunks.
#ifndef HFMM_L2T_V3
#define HFMM_L2T_V3 1
#endif
#ifndef HFMM_L2T_PB
#define HFMM_L2T_PB 4   // points per lane sub-batch (4: 122 registers, 4 CTAs/SM; 8: 164, 3 CTAs/SM)
#endif
template <int PB>
__global__ void __launch_bounds__(SMALL_TPB) l2t_warp3_kernel(PointsDev pts, const int64_t *__restrict__ first,
                                                              const double *__restrict__ cx,
                                                              const double *__restrict__ cy,
                                                              const double *__restrict__ cz, int32_t box0,
                                                              int32_t box1, const double *__restrict__ ks,
                                                              int64_t K, const double2 *__restrict__ L, double w,
                                                              const double *__restrict__ wk,
                                                              double2 *__restrict__ y_far) {
  static_assert(32 % PB == 0, "PB divides the 32-point batch");
  __shared__ double2 tab[TAB];
  __shared__ double wx[SMALL_WARPS][32], wy[SMALL_WARPS][32], wz[SMALL_WARPS][32];
  fill_exp_table(tab);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * SMALL_WARPS;
  const double ws = wk ? 1.0 : w;
  for (int64_t b = box0 + (int64_t)blockIdx.x * SMALL_WARPS + warp; b < box1; b += nwarps) {
    const int64_t s0 = first[b], s1 = first[b + 1];
    const double c0x = cx[b], c0y = cy[b], c0z = cz[b];
    const double2 *Lb = L + b * K;
    for (int64_t j0 = s0; j0 < s1; j0 += 32) {  // batches of 32 points
      const int cnt = (int)min((int64_t)32, s1 - j0);
      __syncwarp();
      {  // c_a - x_i (0 for the unused slots: their sums are discarded)
        const bool v = lane < cnt;
        wx[warp][lane] = v ? c0x - pts.x[j0 + lane] : 0.0;
        wy[warp][lane] = v ? c0y - pts.y[j0 + lane] : 0.0;
        wz[warp][lane] = v ? c0z - pts.z[j0 + lane] : 0.0;
      }
      __syncwarp();
      double yr = 0.0, yi = 0.0;  // lane p: point j0 + p
      for (int p0 = 0; p0 < cnt; p0 += PB) {
        double ar[PB], ai[PB];
#pragma unroll
        for (int p = 0; p < PB; ++p) ar[p] = ai[p] = 0.0;
        for (int64_t k0 = 0; k0 < K; k0 += 32) {
          const int64_t k = k0 + lane;
          const bool v = k < K;
          const double kx = v ? ks[k] : 0.0, ky = v ? ks[K + k] : 0.0, kz = v ? ks[2 * K + k] : 0.0;
          double2 l = v ? Lb[k] : make_double2(0.0, 0.0);
          if (wk) {  // per-point weights (ragged rows, R-15)
            const double wv = v ? wk[k] : 0.0;
            l = make_double2(wv * l.x, wv * l.y);
          }
#pragma unroll
          for (int p = 0; p < PB; ++p) {
            const double dx = wx[warp][p0 + p], dy = wy[warp][p0 + p], dz = wz[warp][p0 + p];
            const double2 e = cexpi_u(fma(kx, dx, fma(ky, dy, kz * dz)), tab);
            ar[p] = fma(e.x, l.x, fma(-e.y, l.y, ar[p]));
            ai[p] = fma(e.x, l.y, fma(e.y, l.x, ai[p]));
          }
        }
#pragma unroll
        for (int p = 0; p < PB; ++p) {
          double pr = ar[p], pi = ai[p];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            pr += __shfl_xor_sync(0xffffffffu, pr, off);
            pi += __shfl_xor_sync(0xffffffffu, pi, off);
          }
          if (lane == p0 + p) yr = pr, yi = pi;
        }
      }
      if (lane < cnt) y_far[j0 + lane] = make_double2(ws * yr, ws * yi);
    }
  }
}

static unsigned persistent_grid(int64_t nbox, const void *fn) {
  int per_sm = 0, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SMALL_TPB, 0);
  const int64_t need = (nbox + SMALL_WARPS - 1) / SMALL_WARPS;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)nsm * std::max(per_sm, 1)));
}

void launch_s2m_small(PointsDev pts, const int64_t *first, const double *cx, const double *cy, const double *cz,
                      int32_t box0, int32_t box1, const double *ks, int64_t K, double2 *M, cudaStream_t s) {
  if (box1 <= box0) return;
  s2m_warp_kernel<<<persistent_grid(box1 - box0, (const void *)s2m_warp_kernel), SMALL_TPB, 0, s>>>(
      pts, first, cx, cy, cz, box0, box1, ks, K, M);
}

void launch_l2t_small(PointsDev pts, const int64_t *first, const double *cx, const double *cy, const double *cz,
                      int32_t box0, int32_t box1, const double *ks, int64_t K, const double2 *L, double w,
                      const double *wk, double2 *y_far, cudaStream_t s) {
  if (box1 <= box0) return;
#if HFMM_L2T_V3
  l2t_warp3_kernel<HFMM_L2T_PB><<<persistent_grid(box1 - box0, (const void *)l2t_warp3_kernel<HFMM_L2T_PB>), SMALL_TPB, 0, s>>>(
      pts, first, cx, cy, cz, box0, box1, ks, K, L, w, wk, y_far);
#elif HFMM_L2T_V2
  l2t_warp2_kernel<<<persistent_grid(box1 - box0, (const void *)l2t_warp2_kernel), SMALL_TPB, 0, s>>>(
      pts, first, cx, cy, cz, box0, box1, ks, K, L, w, wk, y_far);
#else
  l2t_warp_kernel<<<persistent_grid(box1 - box0, (const void *)l2t_warp_kernel), SMALL_TPB, 0, s>>>(
      pts, first, cx, cy, cz, box0, box1, ks, K, L, w, wk, y_far);
#endif
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
    y_out[perm ? perm[i] : i] = a;   // perm == nullptr: keep the sorted order
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
