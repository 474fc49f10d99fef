// Internal declarations of libhfmm (product code; shares nothing with oracle/).
// Citations "P:n" = line n of the paper's LaTeX source.
#pragma once

#include <cstdint>
#include <complex>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace hfmm {

using cplx = std::complex<double>;

// One lock for the process-wide per-device caches (twiddles, __constant__ uploads, operator index
// arrays, device twiddle offsets): concurrent plans on several devices from several threads
// (one thread per GPU) must not race on their std::map / std::set insertions.
std::recursive_mutex &cache_mutex();

// ---------------- host special functions (host_specfun.cpp) ---------------------------------
// Spherical Bessel j_n (Miller, downward), y_n (upward), cylindrical J_n (Miller).
void sph_bessel_j(int nmax, double x, std::vector<double> &out);
void sph_bessel_y(int nmax, double x, std::vector<double> &out);
void cyl_bessel_J(int nmax, double x, std::vector<double> &out);

// ---------------- host plan (host_plan.cpp) -------------------------------------------------
// c_n = (i kappa / 4 pi) i^n (2n+1) h_n(kappa |r0|)  (eqn:TransferFn)
void transfer_series(int ell, double kappa, double r0norm, std::vector<cplx> &c);
// Alg. 1 for one phi column: T^{s,L}(theta_p, phi), p < n_theta.
void alg1_column(int ell, const std::vector<cplx> &c, const double r0hat[3], double phi,
                 int n_theta, std::vector<cplx> &out);
double collino_bound(int ell, double kappa, double r, double r0);
int select_ell(double kappa, double r, double r0, double eps, int *ell);
int select_ntheta(int ell, double kappa, double r, double r0, double eps, int *nth);
int select_nphi(int ell, double kappa, double r, double r0, double eps, int nth, int *nph,
                std::vector<int> *ragged, std::vector<int> *first7 = nullptr);
int select_nphi_rows(int ell, double kappa, double r, double r0, double eps, int nth, int cap,
                     std::vector<int> &rows);  // R-15
bool seven_smooth(int n);
int select_rep_grid(double kappa, double a, double eps, int *nth, int *nph);  // R-14

// ---------------- tree (host_tree.cpp) ------------------------------------------------------
struct LevelBoxes {
  int level = 0;
  double a = 0;
  std::vector<uint32_t> key;       // Morton key of occupied boxes (sorted)
  std::vector<int32_t> ix, iy, iz; // integer coordinates
  std::vector<int64_t> first;      // first sorted point of box, size nbox+1
  std::vector<int32_t> parent;     // index into level l-1 (or -1)
  std::vector<int32_t> child_begin;// children range in level l+1 (size nbox+1), filled lazily
  int64_t nbox() const { return (int64_t)key.size(); }
  int32_t find(int x, int y, int z) const;  // -1 if not occupied
};

struct Tree {
  int64_t n = 0;
  int depth = 0;
  double lo[3] = {0, 0, 0};
  double size = 0;
  std::vector<int64_t> perm;       // sorted position -> input index
  std::vector<double> xs, ys, zs;  // sorted coordinates
  std::vector<LevelBoxes> levels;  // index = level (0..depth)
};

int build_tree(const double *xyz, int64_t n, int depth, const double lo[3], double size, Tree &t,
               std::string &err);
uint32_t morton3(uint32_t x, uint32_t y, uint32_t z);
void partition_level2(const Tree &t, int L_f, int64_t K, int R, std::vector<int64_t> &cut);
void m2l_halo_lists(const Tree &t, int l, const std::vector<int64_t> &rlo, const std::vector<int64_t> &rhi, int r,
                    std::vector<std::vector<int64_t>> &snd, std::vector<std::vector<int64_t>> &rcv);
// offsets: id in [0,316) <-> (ox, oy, oz) in [-3,3]^3 \ [-1,1]^3, lexicographic x, y, z
int offset_id(int ox, int oy, int oz);
void offset_vec(int id, int o[3]);
// NEXT 3: the 34 canonical offsets (x >= y >= 0, z >= 0; cids = their offset ids) and,
// per offset, canonical index << 4 | op with op = x-flip | y-flip << 1 | z-flip << 2 | swap << 3
void canonical_offsets(std::vector<int> &cids, std::vector<int> &sym_of);
// perm[op][k]: stored grid index of the canonical table that holds T_o at stored point k
void symmetry_perms(int nth, int nph, std::vector<int32_t> &perm);

// ---------------- device kernels (kernels_*.cu) ---------------------------------------------
struct ResampleDims {
  int nth, nph;    // source grid
  int nth2, nph2;  // target grid
};

// Longest 1-D transform supported by the resampling kernels (grids N_theta, N_phi < kMaxFFT).
constexpr int kMaxFFT = 4096;
// twiddle table e^{-2 pi i t / N}, t < N, for every length of a plan (device, concatenated)
struct TwiddleSet {
  double2 *d = nullptr;
  int offset[kMaxFFT];  // offset[N] into d, -1 if absent (N < kMaxFFT)
  void build(const std::vector<int> &lengths);
  void free_all();
};

void launch_permute_q(const double2 *q_in, const int64_t *perm, double2 *q_sorted, int64_t n,
                      cudaStream_t s);
// out[(oidx ? oidx[i] : i)][k] = in[(iidx ? iidx[i] : i)][k] for i < count, k < K (M2L halo pack / scatter)
void launch_gather_boxes(const double2 *in, const int64_t *iidx, double2 *out, const int64_t *oidx, int64_t count,
                         int64_t K, cudaStream_t s);
void launch_combine(const double2 *y_near, const double2 *y_far, const int64_t *perm,
                    double2 *y_out, int64_t n, int64_t begin, int64_t end, cudaStream_t s);

struct PointsDev {
  const double *x, *y, *z;  // sorted coordinates
  const double2 *q;         // sorted charges
};

// Positions pre-scaled to table steps (u = x kappa TAB_STEPS / 2 pi) and sorted charges, for P2P.
struct PointsU {
  const double *ux, *uy, *uz;
  const double2 *q;
};
#ifndef HFMM_P2P_MINB
#define HFMM_P2P_MINB 2  // resident CTAs per SM requested from ptxas for 4 targets / thread
#endif
#ifndef HFMM_P2P_TPB
#define HFMM_P2P_TPB 128  // threads per P2P CTA
#endif
constexpr int P2P_THREADS = HFMM_P2P_TPB;
constexpr int P2P_TPB_HOST = HFMM_P2P_TPB;  // work-item tile = P2P_TPB_HOST x targets per thread (3 or 4)
#ifndef HFMM_TAB_STEPS
#define HFMM_TAB_STEPS 2048
#endif
constexpr int TAB_STEPS = HFMM_TAB_STEPS;  // e^{i h k} table size; h = 2 pi / TAB_STEPS
enum { P2P_SYM = 0, P2P_DIAG = 1, P2P_ORD = 2, P2P_DSYM = 3 };
#ifndef HFMM_P2P_DSYM
#define HFMM_P2P_DSYM 1  // matvec diagonal tiles with the symmetric kernel (each unordered pair once)
#endif
// P2P work items, int64 [nitems][4] = (t0, t1, s0, s1): targets [t0, t1) (<= 128 x 3 or 4), sources
// [s0, s1).  P2P_SYM: disjoint ranges, rows and columns (each unordered pair once);
// P2P_DIAG: rows only, self pair masked (sources contain the targets); P2P_ORD: rows only;
// P2P_DSYM (launch kind of the matvec's diagonal tiles, s-range == t-range): symmetric, pairs once.
// Adds scale * sum into y_near (zeroed beforehand); scale = kappa TAB_STEPS / (2 pi).
// dummy_t / dummy_s (scaled units): far positions used to pad partial symmetric tiles.
void launch_p2p_items(PointsU pts, const int64_t *items, int64_t nitems, int kind, double scale,
                      const double dummy_t[3], const double dummy_s[3], double2 *y_near, cudaStream_t s, int pt,
                      double2 *part = nullptr, const int64_t *slot = nullptr, bool rowskip = false);
// deterministic P2P accumulation: y_near[i] = sum of part[idx[e]], e in [row_ptr[i], row_ptr[i + 1])
void launch_p2p_reduce(const double2 *part, const int64_t *row_ptr, const int64_t *idx, int64_t n, double2 *y_near,
                       cudaStream_t s);

// S2M: M[b][k] = sum_j q_j e^{i kappa s_k.(x_j - c_b)}; ks = kappa s / h (table steps)
void launch_s2m(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, int32_t box0, int32_t box1, const double *ks /*[3][K]*/,
                int64_t K, double2 *M, cudaStream_t s);

// L2T: y_far[i] = sum_k w_k L[b][k] e^{i kappa s_k.(c_b - x_i)}; ks as for S2M;
// w_k = wk[k] (ragged rows, R-15) or the constant w
void launch_l2t(PointsDev pts, const int64_t *first, const double *cx, const double *cy,
                const double *cz, const int32_t *tile_leaf, const int64_t *tile_begin,
                int64_t ntiles, const double *ks, int64_t K, const double2 *L, double w,
                const double *wk, double2 *y_far, cudaStream_t s);

// Ragged quadrature (R-15, kernels_ragged.cu): tables from the rectangular ones; 5-step steps 1
// (ragged rows -> rectangular calN_phi half) and 5 (rectangular -> ragged rows), one CTA per row.
void launch_ragged_tables(const double2 *Trect, int ncanon, int nth, int nphr, const int32_t *rows, const int64_t *off,
                          int64_t K, double2 *out, const TwiddleSet &tw, cudaStream_t s);
// item o < nitem: input box par ? par[o] : o of `in` (stride in_K), times conj(shift[oct[o]]) if
// shift; output rectangular half [nth][nphr/2] of box o.
void launch_rag2rect(const double2 *in, int64_t in_K, int nth, const int32_t *rows, const int64_t *off, int maxrow,
                     const int32_t *par, const int8_t *oct, const double2 *shift, int64_t nitem, int nphr,
                     double2 *out, const TwiddleSet &tw, cudaStream_t s);
// item o: sum over children c in [cbeg[o], cbeg[o+1]) (input box c - cbase; c = o without cbeg)
// of shift[oct[c]] (if shift) * (row resample of child c to the ragged rows), + add[o]; into out[o].
void launch_rect2rag(const double2 *in, int nth, int nphr, const int32_t *cbeg, int64_t cbase, const int8_t *oct,
                     const double2 *shift, const double2 *add, const int32_t *rows, const int64_t *off, int64_t K,
                     int64_t nitem, double2 *out, const TwiddleSet &tw, cudaStream_t s);

// Small-box variants (source level below L_f, R-14): one warp per box, persistent grid.
void launch_s2m_small(PointsDev pts, const int64_t *first, const double *cx, const double *cy, const double *cz,
                      int32_t box0, int32_t box1, const double *ks, int64_t K, double2 *M, cudaStream_t s);
void launch_l2t_small(PointsDev pts, const int64_t *first, const double *cx, const double *cy, const double *cz,
                      int32_t box0, int32_t box1, const double *ks, int64_t K, const double2 *L, double w,
                      const double *wk, double2 *y_far, cudaStream_t s);

// Sibling-group M2L (kernels_m2l.cu): plan once per level / operator, apply per matvec.
struct M2LGroupPlan;
// targets = boxes [0, nbox) with host CSR row/src/oid (oid = offset id 0..315); groups
// [gbeg[i], gbeg[i+1]) of <= 8 boxes (nullptr: consecutive blocks of 8)
M2LGroupPlan *m2l_group_plan_create(int64_t nbox, int64_t K, const int32_t *row, const int32_t *src,
                                    const int32_t *oid, const std::vector<int64_t> *gbeg);
void m2l_group_plan_destroy(M2LGroupPlan *pl);
int m2l_group_plan_kind(const M2LGroupPlan *pl);  // 1 parent-block, 0 merged-list, -1 none
// T: [316][K] (perm == nullptr) or the 34 canonical tables [34][K] with perm [16][K]
void m2l_group_apply(const M2LGroupPlan *pl, const double2 *T, const int32_t *perm, const double2 *M, double2 *I,
                     cudaStream_t s);

// Single-pass upward resample (rows + columns of each child on chip) for the small square grids
// it is instantiated for: out[item] = sum_{c in [cbeg[item], cbeg[item+1])} shift[oct[c]] * R(in[c - cbase])
// (cbeg == nullptr: one box per item, no shift).  Returns false when not applicable.
bool box2_up_applies(int nth, int nph, int nth2, int nph2);
bool box2_down_applies(int nth, int nph, int nth2, int nph2);
// Fused two-pass upward resampler (kernels_fused.cu): rows and columns of every item as dependent
// tasks of one persistent kernel, the intermediate in an L2-sized ring (ring = workspace of
// ring_elems complex values, cnt = 2 nitem + 1 ints).  False when not instantiated / disabled
// (HFMM_FUSED=0) or the workspace is too small.
bool fused_enabled();
bool launch_fused_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                     int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, double2 *ring,
                     size_t ring_elems, int *cnt, const TwiddleSet &tw, cudaStream_t s);
// NEXT 4 coefficient-domain symmetric resampling (kernels_sym.cu; opt-in HFMM_NEXT4=1): same
// arguments and result as launch_box2_up / launch_box2_down; false when not enabled or the grid
// pair has no instantiation.
bool next4_enabled();
bool sym2_up_applies(int nth, int nph, int nth2, int nph2);
bool sym2_down_applies(int nth, int nph, int nth2, int nph2);
bool launch_sym2_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, const TwiddleSet &tw,
                    cudaStream_t s);
bool launch_sym2_down(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *par,
                      const int8_t *oct, const double2 *shift, const double2 *add, double2 *out, const TwiddleSet &tw,
                      cudaStream_t s);
bool launch_box2_down(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *par,
                      const int8_t *oct, const double2 *shift, const double2 *add, double2 *out, const TwiddleSet &tw,
                      cudaStream_t s);
bool launch_box2_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, const TwiddleSet &tw,
                    cudaStream_t s);
// Fourier resampling building blocks, warp-per-sequence shared-memory FFTs.
// Row pass of an upward resample: for each box b and row n <= nth/2, full row of length nph
// (stored rows n and (nth-n)%nth) resampled to nph2 -> tmp[b][n][0..nph2).
void launch_rows_up(const double2 *in, int64_t nbox, int nth, int nph, int nph2, double2 *tmp,
                    const TwiddleSet &tw, cudaStream_t s);
// Column pass of an upward resample with child accumulation: for parent p and column
// m < nph2/2: out[p][.][m] = sum_{c in children(p)} shift[oct(c)][.][m] * R_theta(col_c).
// child ids of parent p: [cbeg[p], cbeg[p+1]) (cbeg == nullptr: child p only, shift
// optional), tmp row of child c is c - cbase, oct: child octant (0..7, absolute c) or nullptr.
void launch_cols_up(const double2 *tmp, int nth, int nph2, int nth2, const int32_t *cbeg,
                    int64_t cbase, const int8_t *oct, int64_t nparent, const double2 *shift, double2 *out,
                    const TwiddleSet &tw, cudaStream_t s);
// Column pass of a downward resample: for child c (parent par[c]) and column m < nph/2:
// tmp[c][.][m] = R_theta(conj(shift[oct(c)]) * in[par[c]])[.][m]   (nth -> nth2)
void launch_cols_down(const double2 *in, int nth, int nph, int nth2, const int32_t *par,
                      const int8_t *oct, int64_t nchild, const double2 *shift, double2 *tmp,
                      const TwiddleSet &tw, cudaStream_t s);
// Row pass of a downward resample: rows n <= nth2/2 of tmp (length nph via symmetry),
// resampled to nph2, written to out (half storage) + add (optional).
void launch_rows_down(const double2 *tmp, int64_t nbox, int nth2, int nph, int nph2,
                      const double2 *add, double2 *out, const TwiddleSet &tw, cudaStream_t s);

// Alg. 1 transfer tables on the GPU (precompute).
void launch_alg1_tables(const double2 *coef /*[nr][ell+1]*/, const int32_t *coef_of_offset,
                        const double *r0hat /*[noff][3]*/, int noff, int ell, int nth, int nphf, int qcount,
                        double2 *out /*[noff][nth][qcount]*/, cudaStream_t s);
void launch_phi_anterp(const double2 *full /*[noff][nth][nphf]*/, int noff, int nth, int nphf, int nph,
                       double2 *out /*[noff][nth][nph/2]*/, cudaStream_t s);
void launch_absmax(const double2 *v, int64_t n, double *out /*device, 1 value*/, cudaStream_t s);

}  // namespace hfmm
