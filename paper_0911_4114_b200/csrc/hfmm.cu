// libhfmm C ABI and matvec orchestration (product code, sm_100a).  See include/hfmm.h.
// Pass order of one matvec:
//   permute q -> S2M (L_f) -> M2M (L_f..3) -> [all-gather M_l, multi-GPU] -> M2L (2..L_f)
//   -> L2L (2..L_f-1) -> L2T (L_f) ; P2P (L_f) on a second stream ; combine + unpermute.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX: named host ranges per pass (no-op without a tool)
#include "hfmm_impl.h"
#include "../../include/hfmm.h"

#ifndef HFMM_STREAM_PRIORITY
#define HFMM_STREAM_PRIORITY 1
#endif

using namespace hfmm;

namespace {

const double kPi = 3.14159265358979323846;
const double kURound = 1.1102230246251565e-16;  // 2^-53
const int64_t kTile = 256;                       // targets per L2T tile (2 per thread)

struct LevelDev {
  int l = 0;
  double a = 0;
  int ell = 0, nth = 0, nph = 0;
  double alpha = 0;
  int64_t K = 0;
  double F = NAN;
  bool active = false;
  bool rep = false;              // translation-only level L_f < l <= D_s (R-14)
  bool ragged = false;           // R-15: rows of N_phi(theta_n) points (active levels, HFMM_RAGGED)
  std::vector<int32_t> rows_h;   // N_phi(theta_n), n < nth (ragged)
  std::vector<int64_t> off_h;    // row offsets into the stored half, n <= nth (ragged)
  int32_t *rows_d = nullptr;
  int64_t *off_d = nullptr;
  int64_t K_rect = 0;            // nth * nph / 2 of the rectangular grid (nph = max row)
  double *wk = nullptr;          // per-point L2T weights 8 pi^2 / (nth N_phi(theta_n)) (ragged source level)
  int64_t nbox = 0;
  int64_t own0 = 0, own1 = 0;  // owned box range (Morton order)
  std::vector<int64_t> rlo, rhi; // every rank's owned range (for the all-gather)
  // M2L halo (levels >= HFMM_HALO_LEVEL of a multi-rank plan): instead of the all-gather of M_l,
  // rank r receives from each peer q exactly the q-owned boxes in the interaction lists of its
  // owned boxes (sorted box ids; both sides derive the same lists from the replicated tree)
  bool halo = false;
  std::vector<int64_t> hs_off, hr_off;        // [R + 1] offsets of the send / receive lists by peer
  int64_t *hs_idx = nullptr, *hr_idx = nullptr;  // box ids: sent (owned) / received (peers')
  double2 *hs_buf = nullptr, *hr_buf = nullptr;  // packed [count][K]
  double *cx = nullptr, *cy = nullptr, *cz = nullptr;
  double *ks = nullptr;          // kappa s [3][K]
  double2 *T = nullptr;          // [34][K]: the canonical transfer vectors x >= y >= 0, z >= 0
  int32_t *perm = nullptr;       // [16][K]: grid permutation of each reflection / swap op (NEXT 3)
  double2 *M = nullptr, *I = nullptr, *L = nullptr;  // [nbox][K]
  M2LGroupPlan *m2lg = nullptr;  // sibling-group M2L plan over the owned boxes
  int64_t il_nnz = 0;
  int32_t *parent = nullptr;     // into level l-1
  int8_t *oct = nullptr;         // octant of the box inside its parent
  int32_t *cbeg = nullptr;       // children range into level l+1
  double2 *shift = nullptr;      // [8][K] e^{i kappa s.(c_child - c_parent)} on this grid
};

template <class T>
T *dalloc(size_t count) {
  if (!count) return nullptr;
  void *p = nullptr;
  if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
  return (T *)p;
}

template <class T>
T *dupload(const std::vector<T> &h) {
  if (h.empty()) return nullptr;
  T *d = dalloc<T>(h.size());
  if (d) cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}

TwiddleSet &global_twiddles(int device) {
  std::lock_guard<std::recursive_mutex> lk(cache_mutex());
  static std::map<int, std::unique_ptr<TwiddleSet>> sets;
  auto it = sets.find(device);
  if (it != sets.end()) return *it->second;
  std::vector<int> lens;
  for (int N = 2; N < kMaxFFT; ++N)
    if (seven_smooth(N)) lens.push_back(N);
  auto ts = std::make_unique<TwiddleSet>();
  ts->build(lens);
  TwiddleSet &ref = *ts;
  sets[device] = std::move(ts);
  return ref;
}

}  // namespace

// Virtual ranks (test mode, include/hfmm.h hfmm_vgroup_*): R plans of one process on one device
// act as the ranks of a multi-GPU run; their collectives become one cudaMemcpyAsync per peer
// block between the plans' buffers, driven phase by phase by hfmm_vgroup_matvec.
struct hfmm_vgroup {
  int nranks = 0;
  std::vector<hfmm_plan *> plans;
};

struct hfmm_plan {
  int device = 0;
  cudaStream_t stream = nullptr, stream2 = nullptr, stream_hi = nullptr;  // near field low, far chain high priority
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join_hi = nullptr;
  cudaStream_t stream3 = nullptr;   // second near-field stream (low priority): the <= 384-point tile class
  cudaEvent_t ev_mix = nullptr;     // ... joined into stream2 before the near-field reduction
  cudaEvent_t ev_up = nullptr;   // far chain: M_l of every level up to date (virtual-rank exchange)
  std::string err;
  bool have_tree = false, have_plan = false;
  Tree tree;
  // dist
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  hfmm_vgroup *vg = nullptr;      // virtual ranks in one process (test mode, hfmm_set_dist_virtual)
  std::vector<int64_t> pt_lo, pt_hi;  // every rank's owned sorted point range (y gather)
  double2 *y_sorted = nullptr;    // y in sorted order (multi-rank gather)
  // points (sorted)
  double *px = nullptr, *py = nullptr, *pz = nullptr;
  int64_t *perm = nullptr;
  double2 *q_in = nullptr, *q_sorted = nullptr, *y_out = nullptr, *y_near = nullptr, *y_far = nullptr;
  // plan
  double kappa = 0, eps = 0, alpha = 0, tau = 0;
  unsigned flags = 0;
  int L_f = -1;
  int D_s = -1;              // source level (S2M / L2T), R-14; -1 without far field
  bool small_src = false;    // source boxes small: warp-per-box S2M / L2T kernels
  int64_t *first_src = nullptr;  // point ranges of source-level boxes
  std::vector<LevelDev> lv;  // index = level
  int near_level = 0;        // level of the near-field boxes (L_f or 0)
  int64_t own_pt0 = 0, own_pt1 = 0;
  int64_t *first_near = nullptr;  // point ranges of near-level boxes
  int32_t *tile_leaf = nullptr;    // L2T tiles (kTile targets of one far-field leaf)
  int64_t *tile_begin = nullptr;
  int64_t ntiles = 0;
  // P2P work items [n][4] = (t0, t1, s0, s1) by kind (P2P_SYM, P2P_DIAG, P2P_ORD), and the
  // all-pairs items of hfmm_direct; positions pre-scaled to table steps (kappa-dependent)
  int64_t *p2p_items[3] = {nullptr, nullptr, nullptr};
  int64_t p2p_nitems[3] = {0, 0, 0};
  int64_t p2p_n4[3] = {0, 0, 0};   // mixed tiles: the first p2p_n4[k] items hold 512-point tiles, the rest <= 384
  bool p2p_mix = false;            // 512- and 384-point target tiles mixed per leaf (fewest padded slots)
  int64_t *dir_items = nullptr;
  int64_t dir_nitems = 0;
  double *ux = nullptr, *uy = nullptr, *uz = nullptr;
  double uscale = 0;               // kappa TAB_STEPS / (2 pi)
  int p2p_pt = 4;                  // targets per thread of the P2P kernels (tile = 128 x p2p_pt: 3, 4 or 8)
  bool p2p_rowskip = false;        // symmetric P2P skips dead warp rows (plan: > 8% dead tile slots)
  double p2p_dead_frac = 0.0;      // tile slots of the P2P items holding no live target
  int64_t p2p_sym_pairs = 0;
  double dummy_t[3] = {0, 0, 0}, dummy_s[3] = {0, 0, 0};
  double2 *tmp = nullptr;
  size_t tmp_elems = 0;
  double2 *scr1 = nullptr, *scr2 = nullptr;  // rectangular copies around ragged levels (R-15)
  int *fu_cnt = nullptr;           // task counters of the fused upward resampler (2 max_boxes + 1)
  // deterministic P2P (HFMM_DETERMINISTIC): per-item partial slots, partials, per-point CSR
  int64_t *p2p_slot[3] = {nullptr, nullptr, nullptr};
  double2 *p2p_part = nullptr;
  int64_t *p2p_rp = nullptr, *p2p_idx = nullptr;
  hfmm_info info{};
  double stage_ms[8] = {0};
  bool profile = false;
  cudaEvent_t sev[10] = {nullptr};
};

static thread_local std::string g_create_err;

std::recursive_mutex &hfmm::cache_mutex() {
  static std::recursive_mutex m;
  return m;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      p->err = std::string(#call) + ": " + cudaGetErrorString(e_);                    \
      return HFMM_E_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define CKN(call)                                                                    \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) {                                                         \
      p->err = std::string(#call) + ": " + ncclGetErrorString(r_);                    \
      return HFMM_E_NCCL;                                                            \
    }                                                                                \
  } while (0)
// inside an ncclGroupStart / ncclGroupEnd pair: remember the first failure, keep going so the
// group is always closed (an error return from inside an open group would leave it open)
#define CKG(call)                                                                    \
  do {                                                                               \
    if (gr_ == ncclSuccess) {                                                        \
      gr_ = (call);                                                                  \
      if (gr_ != ncclSuccess) p->err = std::string(#call) + ": " + ncclGetErrorString(gr_); \
    }                                                                                \
  } while (0)

static void free_levels(hfmm_plan *p) {
  for (auto &L : p->lv) {
    m2l_group_plan_destroy(L.m2lg);
    L.m2lg = nullptr;
    for (void *ptr : {(void *)L.cx, (void *)L.cy, (void *)L.cz, (void *)L.ks, (void *)L.T, (void *)L.M,
                      (void *)L.I, (void *)L.L, (void *)L.perm, (void *)L.rows_d, (void *)L.off_d, (void *)L.wk,
                      (void *)L.parent, (void *)L.oct, (void *)L.cbeg, (void *)L.shift, (void *)L.hs_idx,
                      (void *)L.hr_idx, (void *)L.hs_buf, (void *)L.hr_buf})
      if (ptr) cudaFree(ptr);
  }
  p->lv.clear();
  for (void *ptr : {(void *)p->scr1, (void *)p->scr2, (void *)p->first_near, (void *)p->first_src, (void *)p->tile_leaf, (void *)p->tile_begin, (void *)p->tmp,
                    (void *)p->y_far, (void *)p->p2p_items[0], (void *)p->p2p_items[1], (void *)p->p2p_items[2],
                    (void *)p->dir_items, (void *)p->ux, (void *)p->uy, (void *)p->uz, (void *)p->fu_cnt,
                    (void *)p->p2p_slot[0], (void *)p->p2p_slot[1], (void *)p->p2p_slot[2], (void *)p->p2p_part,
                    (void *)p->p2p_rp, (void *)p->p2p_idx})
    if (ptr) cudaFree(ptr);
  p->fu_cnt = nullptr;
  for (auto &q : p->p2p_slot) q = nullptr;
  p->p2p_part = nullptr, p->p2p_rp = p->p2p_idx = nullptr;
  p->first_near = nullptr, p->first_src = nullptr, p->tile_leaf = nullptr;
  p->tile_begin = nullptr, p->tmp = nullptr, p->y_far = nullptr;
  p->scr1 = p->scr2 = nullptr;
  for (int k = 0; k < 3; ++k) p->p2p_items[k] = nullptr, p->p2p_nitems[k] = 0;
  p->dir_items = nullptr, p->dir_nitems = 0;
  p->ux = p->uy = p->uz = nullptr;
  p->tmp_elems = 0;
  p->ntiles = 0;
  p->have_plan = false;
}

static void free_points(hfmm_plan *p) {
  for (void *ptr : {(void *)p->px, (void *)p->py, (void *)p->pz, (void *)p->perm, (void *)p->q_in,
                    (void *)p->q_sorted, (void *)p->y_out, (void *)p->y_near, (void *)p->y_sorted})
    if (ptr) cudaFree(ptr);
  p->px = p->py = p->pz = nullptr;
  p->perm = nullptr;
  p->q_in = p->q_sorted = p->y_out = p->y_near = p->y_sorted = nullptr;
  p->have_tree = false;
}

extern "C" void hfmm_destroy(hfmm_plan *p);

extern "C" int hfmm_create(hfmm_plan **out, int device) {
  if (!out) return HFMM_E_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    g_create_err = "hfmm_create: no CUDA device (libhfmm has no CPU fallback)";
    return HFMM_E_CUDA;
  }
  if (device < 0) cudaGetDevice(&device);
  if (device >= ndev) {
    g_create_err = "hfmm_create: bad device index";
    return HFMM_E_ARG;
  }
  auto *p = new hfmm_plan();
  // on any CUDA failure below: message into g_create_err (what hfmm_last_error(NULL) returns),
  // release what was created, no plan returned
#define CKC(call)                                                                    \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      g_create_err = std::string("hfmm_create: ") + #call + ": " + cudaGetErrorString(e_); \
      hfmm_destroy(p);                                                               \
      return HFMM_E_CUDA;                                                            \
    }                                                                                \
  } while (0)
  p->device = device;
  cudaSetDevice(device);
  CKC(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  {
    // The far-field chain (latency-bound resampling, M2L, S2M/L2T) runs at high priority so its
    // CTAs take SM slots as soon as CTAs of the FP64-bound near field (low priority) retire.
    int lo = 0, hi = 0;
    CKC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
#if HFMM_STREAM_PRIORITY
    CKC(cudaStreamCreateWithPriority(&p->stream2, cudaStreamNonBlocking, lo));
    CKC(cudaStreamCreateWithPriority(&p->stream3, cudaStreamNonBlocking, lo));
    CKC(cudaStreamCreateWithPriority(&p->stream_hi, cudaStreamNonBlocking, hi));
#else
    CKC(cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&p->stream3, cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&p->stream_hi, cudaStreamNonBlocking));
#endif
  }
  CKC(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&p->ev_join_hi, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&p->ev_mix, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&p->ev_up, cudaEventDisableTiming));
  for (auto &e : p->sev) CKC(cudaEventCreate(&e));
  const char *prof = std::getenv("HFMM_PROFILE_STAGES");
  p->profile = prof && prof[0] && prof[0] != '0';
  global_twiddles(device);
  *out = p;
  return HFMM_OK;
#undef CKC
}

extern "C" int hfmm_set_dist(hfmm_plan *p, int rank, int nranks, const void *id) {
  if (!p) return HFMM_E_ARG;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !id)) {
    p->err = "hfmm_set_dist: bad rank/nranks/id";
    return HFMM_E_ARG;
  }
  if (p->have_tree) {
    p->err = "hfmm_set_dist: must be called before build_tree";
    return HFMM_E_STATE;
  }
  cudaSetDevice(p->device);
  if (p->comm) {
    ncclCommDestroy(p->comm);
    p->comm = nullptr;
  }
  p->rank = rank;
  p->nranks = nranks;
  if (nranks > 1) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    CKN(ncclCommInitRank(&p->comm, nranks, uid, rank));
  }
  return HFMM_OK;
}

extern "C" int hfmm_nccl_unique_id(void *out) {
  if (!out) return HFMM_E_ARG;
  ncclUniqueId uid;
  if (ncclGetUniqueId(&uid) != ncclSuccess) return HFMM_E_NCCL;
  std::memcpy(out, &uid, sizeof(uid));
  return HFMM_OK;
}

extern "C" int hfmm_build_tree(hfmm_plan *p, int64_t n, const double *xyz, int depth, const double lo[3],
                               double size) {
  if (!p) return HFMM_E_ARG;
  if (!xyz || !lo) {
    p->err = "hfmm_build_tree: NULL pointer";
    return HFMM_E_ARG;
  }
  cudaSetDevice(p->device);
  free_levels(p);
  free_points(p);
  int rc = build_tree(xyz, n, depth, lo, size, p->tree, p->err);
  if (rc) return rc;
  const Tree &t = p->tree;
  p->px = dupload(t.xs), p->py = dupload(t.ys), p->pz = dupload(t.zs);
  p->perm = dupload(t.perm);
  p->q_in = dalloc<double2>(n), p->q_sorted = dalloc<double2>(n);
  p->y_out = dalloc<double2>(n), p->y_near = dalloc<double2>(n);
  if (p->nranks > 1) p->y_sorted = dalloc<double2>(n);
  if (!p->px || !p->py || !p->pz || !p->perm || !p->q_in || !p->q_sorted || !p->y_out || !p->y_near ||
      (p->nranks > 1 && !p->y_sorted)) {
    p->err = "hfmm_build_tree: device allocation failed";
    return HFMM_E_NOMEM;
  }
  p->have_tree = true;
  return HFMM_OK;
}

// ---- precompute helpers ---------------------------------------------------------------------
static int level_tables(hfmm_plan *p, LevelDev &L, double2 **T_out, double *F_out) {
  // Alg. 1 for the 34 canonical offsets on the GPU; c_n per distinct |r0| from the host.
  std::vector<int> cids, sym_of;
  canonical_offsets(cids, sym_of);
  const int NC = (int)cids.size();
  std::vector<double2> coef;
  std::vector<int32_t> coef_of(NC);
  std::vector<double> r0hat(NC * 3);
  std::map<int, int> by_norm2;
  for (int ci = 0; ci < NC; ++ci) {
    const int id = ci;  // row of the canonical table set
    int o[3];
    offset_vec(cids[ci], o);
    int n2 = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
    auto it = by_norm2.find(n2);
    if (it == by_norm2.end()) {
      std::vector<cplx> c;
      transfer_series(L.ell, p->kappa, std::sqrt((double)n2) * L.a, c);
      int idx = (int)by_norm2.size();
      by_norm2[n2] = idx;
      for (auto &v : c) coef.push_back(make_double2(v.real(), v.imag()));
      coef_of[id] = idx;
    } else {
      coef_of[id] = it->second;
    }
    double nr = std::sqrt((double)n2);
    for (int d = 0; d < 3; ++d) r0hat[3 * id + d] = o[d] / nr;
  }
  for (auto &v : coef)
    if (!std::isfinite(v.x) || !std::isfinite(v.y)) {
      // h_n overflow: deep in the low-frequency breakdown; table unusable
      *T_out = nullptr;
      *F_out = INFINITY;
      return HFMM_OK;
    }
  double2 *dcoef = dupload(coef);
  int32_t *dcof = dupload(coef_of);
  double *dr0 = dupload(r0hat);
  double2 *T = dalloc<double2>((size_t)NC * L.K);
  if (!dcoef || !dcof || !dr0 || !T) {
    p->err = "precompute: allocation failed (transfer tables)";
    return HFMM_E_NOMEM;
  }
  if (L.nph >= 2 * L.ell + 2) {
    launch_alg1_tables(dcoef, dcof, dr0, NC, L.ell, L.nth, L.nph, L.nph / 2, T, p->stream);
  } else {
    const int nphf = 2 * L.ell + 2;
    double2 *full = dalloc<double2>((size_t)NC * L.nth * nphf);
    if (!full) {
      p->err = "precompute: allocation failed (phi-fine tables)";
      return HFMM_E_NOMEM;
    }
    launch_alg1_tables(dcoef, dcof, dr0, NC, L.ell, L.nth, nphf, nphf, full, p->stream);
    launch_phi_anterp(full, NC, L.nth, nphf, L.nph, T, p->stream);
    CK(cudaStreamSynchronize(p->stream));
    cudaFree(full);
  }
  double *dmax = dalloc<double>(1);
  launch_absmax(T, (int64_t)NC * L.K, dmax, p->stream);  // = max over all 316 (reflections)
  double mx = 0;
  CK(cudaMemcpyAsync(&mx, dmax, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  CK(cudaGetLastError());
  cudaFree(dmax);
  cudaFree(dcoef);
  cudaFree(dcof);
  cudaFree(dr0);
  *T_out = T;
  *F_out = 8.0 * kPi * kURound * L.a * mx;
  return HFMM_OK;
}

// kappa s at the stored points, row by row (rows[n] points on row n of a ragged level, R-15;
// nph on every row otherwise): k = off[n] + m, phi = 2 pi m / N_phi(theta_n), m < N_phi(theta_n)/2
static void grid_dirs(const LevelDev &L, double kappa, std::vector<double> &ks) {
  const int64_t K = L.K;
  ks.assign(3 * K, 0.0);
  int64_t k = 0;
  for (int n = 0; n < L.nth; ++n) {
    long double th = 2.0L * 3.141592653589793238462643383279502884L * n / L.nth;
    double st = (double)sinl(th), ct = (double)cosl(th);
    const int nph = L.ragged ? L.rows_h[n] : L.nph;
    for (int m = 0; m < nph / 2; ++m, ++k) {
      long double ph = 2.0L * 3.141592653589793238462643383279502884L * m / nph;
      double cp = (double)cosl(ph), sp = (double)sinl(ph);
      ks[k] = kappa * (cp * st);
      ks[K + k] = kappa * (sp * st);
      ks[2 * K + k] = kappa * ct;
    }
  }
}

// perm[op][k] of the 34-table reflections on a ragged grid (row-local phi maps; row lengths are
// symmetric under theta -> pi - theta and theta -> 2 pi - theta, R-15)
static void symmetry_perms_ragged(const LevelDev &L, std::vector<int32_t> &perm) {
  const int nth = L.nth;
  perm.assign((size_t)16 * L.K, 0);
  for (int op = 0; op < 16; ++op)
    for (int n = 0; n < nth; ++n) {
      const int N = L.rows_h[n];
      for (int m = 0; m < N / 2; ++m) {
        int nn = n, mm = m;
        if (op & 1) mm = (N / 2 - mm + N) % N;
        if (op & 2) mm = (N - mm) % N;
        if (op & 4) nn = (nth / 2 - nn + nth) % nth;
        if (op & 8) mm = ((N / 4 - mm) % N + N) % N;
        if (mm >= N / 2) nn = (nth - nn) % nth, mm -= N / 2;
        perm[(size_t)op * L.K + L.off_h[n] + m] = (int32_t)(L.off_h[nn] + mm);
      }
    }
}

// Levels l >= this exchange M2L halos instead of all-gathering M_l (multi-rank plans).  Default 4:
// the coarse top levels (2, 3) are replicated by the all-gather; read at every
// precompute so a test can move it (HFMM_HALO_LEVEL=2: every active level as halos).
static int halo_min_level() {
  const char *e = getenv("HFMM_HALO_LEVEL");
  return e ? atoi(e) : 4;
}

static void partition(hfmm_plan *p) {
  // Ownership by contiguous Morton ranges of level-2 subtrees (or of points if no far field),
  // balanced by an estimate of FP64 work: P2P pairs + S2M/L2T evaluations.  Every rank
  // computes every rank's ranges (needed for the variable-size all-gather).
  const Tree &t = p->tree;
  const int R = p->nranks, r = p->rank;
  if (p->L_f < 0) {
    const int64_t n = t.n;
    auto cutp = [&](int k) -> int64_t {
      if (k >= R) return n;
      int64_t c = (n * k / R) / kTile * kTile;   // tile-aligned (P2P tiles are kTile targets)
      return std::min(c, n);
    };
    p->own_pt0 = cutp(r);
    p->own_pt1 = cutp(r + 1);
    p->pt_lo.assign(R, 0), p->pt_hi.assign(R, 0);
    for (int q = 0; q < R; ++q) p->pt_lo[q] = cutp(q), p->pt_hi[q] = cutp(q + 1);
    return;
  }
  const LevelBoxes &BL = t.levels[p->L_f];
  std::vector<int64_t> cut;
  partition_level2(t, p->L_f, p->lv[p->L_f].K, R, cut);
  for (int l = 2; l <= std::max(p->L_f, p->D_s); ++l) {
    LevelDev &L = p->lv[l];
    L.rlo.assign(R, 0), L.rhi.assign(R, 0);
    for (int q = 0; q < R; ++q) {
      if (l == 2) {
        L.rlo[q] = cut[q], L.rhi[q] = cut[q + 1];
      } else {
        const LevelBoxes &P = t.levels[l - 1];
        const LevelDev &U = p->lv[l - 1];
        L.rlo[q] = P.child_begin[U.rlo[q]];
        L.rhi[q] = P.child_begin[U.rhi[q]];
      }
    }
    L.own0 = L.rlo[r], L.own1 = L.rhi[r];
  }
  const LevelDev &Lf = p->lv[p->L_f];
  p->own_pt0 = BL.first[Lf.own0];
  p->own_pt1 = BL.first[Lf.own1];
  p->pt_lo.assign(R, 0), p->pt_hi.assign(R, 0);
  for (int q = 0; q < R; ++q) p->pt_lo[q] = BL.first[Lf.rlo[q]], p->pt_hi[q] = BL.first[Lf.rhi[q]];
}

extern "C" int hfmm_precompute(hfmm_plan *p, double kappa, double eps, double alpha, double tau,
                               unsigned flags) {
  if (!p) return HFMM_E_ARG;
  if (!p->have_tree) {
    p->err = "hfmm_precompute: build_tree first";
    return HFMM_E_STATE;
  }
  if (!(kappa > 0) || !std::isfinite(kappa) || !(eps > 0) || !(eps < 1) || !(alpha > 0) || alpha > 1) {
    p->err = "hfmm_precompute: need kappa > 0, 0 < eps < 1, 0 < alpha <= 1";
    return HFMM_E_ARG;
  }
  cudaSetDevice(p->device);
  free_levels(p);
  p->kappa = kappa, p->eps = eps, p->alpha = alpha, p->flags = flags;
  p->tau = (tau > 0) ? tau : std::min(eps / 10.0, 1e-9);
  const Tree &t = p->tree;
  const int D = t.depth;
  p->lv.assign(D + 1, LevelDev());
  // per-level quadrature (host) for a design radius alpha sqrt(3) a_l
  auto level_quad = [&](LevelDev &L, double al) -> int {
    const double eps_l = (flags & HFMM_EPS_ABSOLUTE) ? eps : eps / L.a;
    const double r = al * std::sqrt(3.0) * L.a, r0 = 2.0 * L.a;
    int rc = select_ell(kappa, r, r0, eps_l, &L.ell);
    if (!rc) rc = select_ntheta(L.ell, kappa, r, r0, eps_l, &L.nth);
    if (!rc) rc = select_nphi(L.ell, kappa, r, r0, eps_l, L.nth, &L.nph, nullptr);
    if (rc) p->err = "hfmm_precompute: quadrature search failed at level " + std::to_string(L.l);
    L.alpha = al;
    L.K = (int64_t)L.nth * L.nph / 2;
    return rc;
  };
  // candidate design radii: the largest alpha in {1, 0.9, 0.8} (>= the caller's alpha) that
  // keeps the level admissible (R-13); the caller's alpha alone with HFMM_ALPHA_FIXED
  std::vector<double> cands;
  if (flags & (HFMM_ALPHA_FIXED | HFMM_FORCE_ALL_LEVELS)) {
    cands.push_back(alpha);
  } else {
    for (double c : {1.0, 0.9, 0.8})
      if (c > alpha + 1e-12) cands.push_back(c);
    cands.push_back(alpha);
  }
  for (int l = 2; l <= D; ++l) {
    LevelDev &L = p->lv[l];
    L.l = l;
    L.a = t.size / (double)(1 << l);
    L.nbox = t.levels[l].nbox();
  }
  // admissibility F_l <= tau, shallowest first (R-9)
  p->L_f = -1;
  const bool force = flags & HFMM_FORCE_ALL_LEVELS;
  int first_inactive = D + 1;
  for (int l = 2; l <= D; ++l) {
    LevelDev &L = p->lv[l];
    for (double al : cands) {
      int rc = level_quad(L, al);
      if (rc) return rc;
      double2 *T = nullptr;
      rc = level_tables(p, L, &T, &L.F);
      if (rc) return rc;
      if (!T && force) {  // h_n overflow: no usable table even when every level is forced
        p->err = "hfmm_precompute: transfer function overflows (h_n) at level " + std::to_string(l) +
                 " -- cannot force it active";
        return HFMM_E_SEARCH;
      }
      L.active = T && (force || (L.F <= p->tau));
      if (L.active) {
        L.T = T;
        break;
      }
      if (T) cudaFree(T);
    }
    if (!L.active) {
      first_inactive = l;
      break;
    }
    p->L_f = l;
  }
  for (int l = first_inactive + 1; l <= D; ++l) {  // reported only (caller's alpha, F not evaluated)
    int rc = level_quad(p->lv[l], alpha);
    if (rc) return rc;
  }
  // source level D_s and the translation-only levels L_f < l <= D_s (R-14)
  p->D_s = -1;
  if (p->L_f >= 2) {
    int Ds = p->L_f;
    if (flags & HFMM_SOURCE_AT_DEPTH) {
      Ds = D;
    } else if (!(flags & HFMM_SOURCE_AT_LF)) {
      for (int l = D; l > p->L_f; --l)
        if ((double)t.n / (double)t.levels[l].nbox() >= 8.0) {
          Ds = l;
          break;
        }
    }
    for (int l = p->L_f + 1; l <= Ds; ++l) {
      LevelDev &L = p->lv[l];
      if (select_rep_grid(kappa, L.a, eps, &L.nth, &L.nph)) {
        p->err = "hfmm_precompute: representation grid search failed at level " + std::to_string(l);
        return HFMM_E_SEARCH;
      }
      L.rep = true, L.active = false, L.ell = 0, L.F = NAN, L.alpha = alpha;
      L.K = (int64_t)L.nth * L.nph / 2;
    }
    p->D_s = Ds;
  }
  // monotone grids along the chain 2..D_s (R-5)
  for (int l = p->D_s - 1; l >= 2; --l) {
    LevelDev &U = p->lv[l], &Dn = p->lv[l + 1];
    int nth = std::max(U.nth, Dn.nth), nph = std::max(U.nph, Dn.nph);
    if (nth != U.nth || nph != U.nph) {
      U.nth = nth, U.nph = nph, U.K = (int64_t)nth * nph / 2;
      if (!U.rep) {
        cudaFree(U.T);
        int rc = level_tables(p, U, &U.T, &U.F);
        if (rc) return rc;
        if (!U.T) {
          p->err = "hfmm_precompute: transfer function overflows (h_n) at level " + std::to_string(l) +
                   " after the monotone-grid rebuild";
          return HFMM_E_SEARCH;
        }
      }
    }
  }
  partition(p);
  // ragged rows on the active levels (R-15), their tables from the rectangular ones
  if ((flags & HFMM_RAGGED) && p->L_f >= 2) {
    const TwiddleSet &tw = global_twiddles(p->device);
    for (int l = 2; l <= p->L_f; ++l) {
      LevelDev &L = p->lv[l];
      const double eps_l = (flags & HFMM_EPS_ABSOLUTE) ? eps : eps / L.a;
      std::vector<int> rows;
      if (select_nphi_rows(L.ell, kappa, L.alpha * std::sqrt(3.0) * L.a, 2.0 * L.a, eps_l, L.nth, L.nph, rows)) {
        p->err = "hfmm_precompute: ragged row search failed at level " + std::to_string(l);
        return HFMM_E_SEARCH;
      }
      L.ragged = true;
      L.rows_h.assign(rows.begin(), rows.end());
      L.off_h.assign(L.nth + 1, 0);
      for (int n = 0; n < L.nth; ++n) L.off_h[n + 1] = L.off_h[n] + rows[n] / 2;
      L.K_rect = (int64_t)L.nth * L.nph / 2;
      L.K = L.off_h[L.nth];
      L.rows_d = dupload(L.rows_h), L.off_d = dupload(L.off_h);
      std::vector<int> cids, sym_of;
      canonical_offsets(cids, sym_of);
      double2 *Tr = dalloc<double2>((size_t)cids.size() * L.K);
      if (!Tr || !L.rows_d || !L.off_d) {
        p->err = "hfmm_precompute: allocation failed (ragged tables)";
        return HFMM_E_NOMEM;
      }
      launch_ragged_tables(L.T, (int)cids.size(), L.nth, L.nph, L.rows_d, L.off_d, L.K, Tr, tw, p->stream);
      CK(cudaStreamSynchronize(p->stream));
      cudaFree(L.T);
      L.T = Tr;
    }
  }
  for (int l = 2; l <= p->D_s; ++l)
    if (p->lv[l].nth >= kMaxFFT || p->lv[l].nph >= kMaxFFT) {
      p->err = "hfmm_precompute: level " + std::to_string(l) + " grid " + std::to_string(p->lv[l].nth) + " x " +
               std::to_string(p->lv[l].nph) + " exceeds the resampling kernels' limit (" + std::to_string(kMaxFFT) + ")";
      return HFMM_E_SEARCH;
    }
  // device data of the levels 2..D_s (M2L data only on the active levels 2..L_f)
  size_t tmp_need = 0, scr1_need = 0, scr2_need = 0;
  for (int l = 2; l <= p->D_s; ++l) {
    LevelDev &L = p->lv[l];
    const LevelBoxes &B = t.levels[l];
    std::vector<double> cx(B.nbox()), cy(B.nbox()), cz(B.nbox());
    for (int64_t b = 0; b < B.nbox(); ++b) {
      cx[b] = t.lo[0] + (B.ix[b] + 0.5) * L.a;
      cy[b] = t.lo[1] + (B.iy[b] + 0.5) * L.a;
      cz[b] = t.lo[2] + (B.iz[b] + 0.5) * L.a;
    }
    L.cx = dupload(cx), L.cy = dupload(cy), L.cz = dupload(cz);
    std::vector<double> ks;
    grid_dirs(L, kappa, ks);
    {
      std::vector<double> ksu(ks);  // kernels take kappa s in table steps (h = 2 pi / TAB_STEPS)
      for (auto &v : ksu) v *= (double)TAB_STEPS / (2.0 * kPi);
      L.ks = dupload(ksu);
    }
    L.M = dalloc<double2>((size_t)L.nbox * L.K);
    L.I = L.active ? dalloc<double2>((size_t)L.nbox * L.K) : nullptr;
    L.L = dalloc<double2>((size_t)L.nbox * L.K);
    if (!L.M || (L.active && !L.I) || !L.L || !L.ks) {
      p->err = "hfmm_precompute: allocation failed (level buffers)";
      return HFMM_E_NOMEM;
    }
    // interaction lists for every box of an active level
    std::vector<int32_t> row(1, 0), src, oid316;
    for (int64_t b = 0; b < (L.active ? B.nbox() : 0); ++b) {
      const int px = B.ix[b] >> 1, py = B.iy[b] >> 1, pz = B.iz[b] >> 1;
      for (int dx = -3; dx <= 3; ++dx)
        for (int dy = -3; dy <= 3; ++dy)
          for (int dz = -3; dz <= 3; ++dz) {
            if (std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz))) < 2) continue;
            int x = B.ix[b] + dx, y = B.iy[b] + dy, z = B.iz[b] + dz;
            if (std::abs((x >> 1) - px) > 1 || std::abs((y >> 1) - py) > 1 || std::abs((z >> 1) - pz) > 1)
              continue;
            int32_t k = B.find(x, y, z);
            if (k < 0) continue;
            src.push_back(k);
            oid316.push_back(offset_id(dx, dy, dz));
          }
      row.push_back((int32_t)src.size());
    }
    L.il_nnz = (int64_t)src.size();
    if (L.active && p->nranks > 1 && l >= halo_min_level()) {
      // halo lists (host_tree.cpp m2l_halo_lists, also exported as hfmm_halo_lists)
      const int R = p->nranks;
      std::vector<std::vector<int64_t>> snd, rcv;
      m2l_halo_lists(t, l, L.rlo, L.rhi, p->rank, snd, rcv);
      L.hs_off.assign(R + 1, 0), L.hr_off.assign(R + 1, 0);
      std::vector<int64_t> hs, hr;
      for (int q = 0; q < R; ++q) {
        hs.insert(hs.end(), snd[q].begin(), snd[q].end());
        hr.insert(hr.end(), rcv[q].begin(), rcv[q].end());
        L.hs_off[q + 1] = (int64_t)hs.size(), L.hr_off[q + 1] = (int64_t)hr.size();
      }
      L.halo = true;
      L.hs_idx = dupload(hs), L.hr_idx = dupload(hr);
      L.hs_buf = dalloc<double2>(hs.size() * (size_t)L.K);
      L.hr_buf = dalloc<double2>(hr.size() * (size_t)L.K);
      if ((!hs.empty() && (!L.hs_idx || !L.hs_buf)) || (!hr.empty() && (!L.hr_idx || !L.hr_buf))) {
        p->err = "hfmm_precompute: allocation failed (M2L halo buffers)";
        return HFMM_E_NOMEM;
      }
    }
    if (L.active) {
      std::vector<int32_t> pm;
      if (L.ragged) symmetry_perms_ragged(L, pm);
      else symmetry_perms(L.nth, L.nph, pm);
      L.perm = dupload(pm);
      // sibling groups over the owned boxes: consecutive boxes (Morton order) with one parent
      std::vector<int64_t> gb;
      for (int64_t b = L.own0; b < L.own1; ++b)
        if (gb.empty() || B.parent[b] != B.parent[b - 1] || b - gb.back() == 8) gb.push_back(b);
      gb.push_back(L.own1);
      if (L.own1 > L.own0) L.m2lg = m2l_group_plan_create(B.nbox(), L.K, row.data(), src.data(), oid316.data(), &gb);
    }
    // tree links
    std::vector<int32_t> par(B.parent.begin(), B.parent.end());
    std::vector<int8_t> oc(B.nbox());
    for (int64_t b = 0; b < B.nbox(); ++b) oc[b] = (int8_t)(((B.ix[b] & 1) << 2) | ((B.iy[b] & 1) << 1) | (B.iz[b] & 1));
    L.parent = dupload(par);
    L.oct = dupload(oc);
    if (l < p->D_s) {
      std::vector<int32_t> cb(B.child_begin.begin(), B.child_begin.end());
      L.cbeg = dupload(cb);
      // translation tables on this grid for children at level l+1
      const double h = 0.5 * p->lv[l + 1].a;
      std::vector<double2> sh((size_t)8 * L.K);
      for (int o = 0; o < 8; ++o) {
        const double d0 = ((o >> 2) & 1) ? h : -h, d1 = ((o >> 1) & 1) ? h : -h, d2 = (o & 1) ? h : -h;
        for (int64_t k = 0; k < L.K; ++k) {
          double ph = ks[k] * d0 + ks[L.K + k] * d1 + ks[2 * L.K + k] * d2;
          sh[(size_t)o * L.K + k] = make_double2(std::cos(ph), std::sin(ph));
        }
      }
      L.shift = dupload(sh);
      const LevelDev &C = p->lv[l + 1];
      tmp_need = std::max(tmp_need, (size_t)C.nbox * (C.nth / 2 + 1) * L.nph);  // M2M rows pass
      tmp_need = std::max(tmp_need, (size_t)C.nbox * C.nth * (L.nph / 2));      // L2L cols pass
      if (C.ragged || L.ragged) {  // rectangular copies: children on the child / parent grids
        scr1_need = std::max(scr1_need, (size_t)C.nbox * C.nth * (C.nph / 2));
        scr2_need = std::max(scr2_need, (size_t)C.nbox * L.nth * (L.nph / 2));
      }
    }
  }
  {
    int64_t maxb = 1;
    for (int l = 2; l <= std::max(p->L_f, p->D_s); ++l) maxb = std::max<int64_t>(maxb, p->lv[l].nbox);
    p->fu_cnt = dalloc<int>((size_t)(2 * maxb + 1));
  }
  if (tmp_need) {
    p->tmp = dalloc<double2>(tmp_need);
    p->tmp_elems = tmp_need;
    if (!p->tmp) {
      p->err = "hfmm_precompute: allocation failed (resample scratch)";
      return HFMM_E_NOMEM;
    }
  }
  if (scr1_need) p->scr1 = dalloc<double2>(scr1_need);
  if (scr2_need) p->scr2 = dalloc<double2>(scr2_need);
  if ((scr1_need && !p->scr1) || (scr2_need && !p->scr2)) {
    p->err = "hfmm_precompute: allocation failed (ragged scratch)";
    return HFMM_E_NOMEM;
  }
  if (p->D_s >= 2 && p->lv[p->D_s].ragged) {  // per-point L2T weights on a ragged source level
    const LevelDev &S = p->lv[p->D_s];
    std::vector<double> w(S.K);
    for (int n = 0; n < S.nth; ++n)
      for (int64_t k = S.off_h[n]; k < S.off_h[n + 1]; ++k) w[k] = 8.0 * kPi * kPi / ((double)S.nth * S.rows_h[n]);
    p->lv[p->D_s].wk = dupload(w);
  }
  // near field at L_f (neighbour lists) or all pairs at the root, as P2P work items
  p->near_level = p->L_f >= 2 ? p->L_f : 0;
  {
    const LevelBoxes &B = t.levels[p->near_level];
    const double kTwoPi = 2.0 * kPi;
    p->uscale = kappa * (double)TAB_STEPS / kTwoPi;
    std::vector<double> ux(t.n), uy(t.n), uz(t.n);
    for (int64_t i = 0; i < t.n; ++i)
      ux[i] = t.xs[i] * p->uscale, uy[i] = t.ys[i] * p->uscale, uz[i] = t.zs[i] * p->uscale;
    p->ux = dupload(ux), p->uy = dupload(uy), p->uz = dupload(uz);
    // Owned target ranges: owned near-level boxes (far field), or the rank's point range of the
    // root (no far field).  Every target tile (<= `tile` points of one box) gets
    //   DIAG (tile, tile);  SYM (tile, later tile of the same box);
    //   SYM (tile, owned neighbour box beta > alpha);  ORD (tile, neighbour range owned elsewhere).
    std::vector<int64_t> it[3];
    int64_t pairs = 0, sym_pairs = 0;
    int64_t tile = (int64_t)P2P_TPB_HOST * 4;   // targets per item: 128 threads x PT targets
    bool mix_tiles = false;
    // per-slot cost of the 384-point kernel relative to the 512-point one (HFMM_P2P_MIX3COST: A/B)
    const double kMix3Cost = getenv("HFMM_P2P_MIX3COST") ? atof(getenv("HFMM_P2P_MIX3COST")) : 1.08;
    auto add = [&](int kind, int64_t t0, int64_t t1, int64_t s0, int64_t s1) {
      if (t1 <= t0 || s1 <= s0) return;
      it[kind].insert(it[kind].end(), {t0, t1, s0, s1});
    };
    auto own_box = [&](int64_t A0, int64_t A1, const std::vector<std::pair<int64_t, int64_t>> &others_owned,
                       const std::vector<std::pair<int64_t, int64_t>> &others_foreign) {
      // targets [A0, A1) of one owned box; others_* = neighbour ranges (sym: only beta > alpha)
      // tile boundaries of the box: fixed tiles, or (mix_tiles) a full 512-point tiles followed by
      // b tiles of <= 384 points, (a, b) minimising the padded slots 512 a + kMix3Cost 384 b
      std::vector<int64_t> cut{A0};
      if (!mix_tiles) {
        for (int64_t t0 = A0; t0 < A1; t0 += tile) cut.push_back(std::min(t0 + tile, A1));
      } else {
        const int64_t nA = A1 - A0, T4 = (int64_t)P2P_TPB_HOST * 4, T3 = (int64_t)P2P_TPB_HOST * 3;
        int64_t ba = 0, bb = 0;
        double best = 1e300;
        for (int64_t a = 0; a <= (nA + T4 - 1) / T4; ++a) {
          const int64_t rest = std::max<int64_t>(0, nA - a * T4), b = (rest + T3 - 1) / T3;
          const double c = (double)(a * T4) + kMix3Cost * (double)(b * T3);
          if (c < best) best = c, ba = a, bb = b;
        }
        int64_t t0 = A0;
        for (int64_t a = 0; a < ba && t0 < A1; ++a) t0 = std::min(t0 + T4, A1), cut.push_back(t0);
        for (int64_t b = 0; b < bb && t0 < A1; ++b) t0 = std::min(t0 + T3, A1), cut.push_back(t0);
      }
      for (size_t c = 0; c + 1 < cut.size(); ++c) {
        const int64_t t0 = cut[c], t1 = cut[c + 1];
        add(P2P_DIAG, t0, t1, t0, t1);
        for (size_t d = c + 1; d + 1 < cut.size(); ++d) add(P2P_SYM, t0, t1, cut[d], cut[d + 1]);
        for (auto &r : others_owned) add(P2P_SYM, t0, t1, r.first, r.second);
        for (auto &r : others_foreign) add(P2P_ORD, t0, t1, r.first, r.second);
      }
    };
    auto build_items = [&]() {
    for (auto &v : it) v.clear();
    pairs = 0;
    if (p->L_f >= 2) {
      const int64_t lo = p->lv[p->L_f].own0, hi = p->lv[p->L_f].own1;
      for (int64_t b = lo; b < hi; ++b) {
        std::vector<std::pair<int64_t, int64_t>> ow, fo;
        const int64_t nb = B.first[b + 1] - B.first[b];
        for (int dx = -1; dx <= 1; ++dx)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dz = -1; dz <= 1; ++dz) {
              int32_t k = B.find(B.ix[b] + dx, B.iy[b] + dy, B.iz[b] + dz);
              if (k < 0) continue;
              const int64_t nk = B.first[k + 1] - B.first[k];
              pairs += nb * nk - (k == b ? nb : 0);
              if (k == b) continue;
              if (k < lo || k >= hi) {
                fo.push_back({B.first[k], B.first[k + 1]});
              } else if (k > b) {
                ow.push_back({B.first[k], B.first[k + 1]});
              }
            }
        own_box(B.first[b], B.first[b + 1], ow, fo);
      }
    } else {
      const int64_t A0 = p->own_pt0, A1 = p->own_pt1, n = t.n;
      std::vector<std::pair<int64_t, int64_t>> fo;
      if (A0 > 0) fo.push_back({0, A0});
      if (A1 < n) fo.push_back({A1, n});
      own_box(A0, A1, {}, fo);
      pairs = (A1 - A0) * (n - 1);
    }
    };
    // Per-plan tile (load balance): 4 targets per thread (512-point tiles, 3 CTAs / SM) unless
    // that leaves fewer than ~10 waves of items over the GPU, or the leaves fill 512-point tiles
    // poorly (padded slots below), then 3 per thread (384-point tiles, 4 CTAs / SM): the tail of
    // a short grid costs more than the slightly lower per-item rate (C3: 11% faster; C4 / C5 keep
    // 512, same-box A/B profiles/r01/p2p_occupancy_ab_r26.txt).
    // HFMM_P2P_PT = 3 / 4 / 8 forces a tile (A/B).  8 targets per thread (1,024-point tiles, 2
    // CTAs / SM) needs fewer FP64 issue slots per evaluation (37.4 vs 38.7 by
    // tools/sass_fp64_cost.py, +3.4% on the uniform-item rig profiles/r02/p2p_ablate2.txt) but is
    // slower on the matvec configs (C4 71.8 vs 68.1 ms, C5 851 vs 758 ms,
    // profiles/r02/pt_ab.txt): opt-in only.
    {
      int nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device);
      int force = 0;
      if (const char *e = getenv("HFMM_P2P_PT")) force = atoi(e);
      const int cand[3] = {8, 4, 3}, ctas[3] = {2, 3, 4};
      // thread-evaluation slots of the items against the sources padded to 32: every thread of a
      // tile evaluates its PT targets (inactive ones at a dummy position), or -- live_only -- only
      // the 32-target warp rows holding a live target (the row-skipping kernel)
      auto padded_slots = [&](int pt, bool live_only = false) {
        double sl = 0.0;
        for (auto &v : it)
          for (size_t i = 0; i < v.size(); i += 4) {
            const int ptm = mix_tiles ? (v[i + 1] - v[i] > 3 * (int64_t)P2P_TPB_HOST ? 4 : 3) : pt;
            const double rows = live_only ? (double)((v[i + 1] - v[i] + 31) / 32 * 32) : (double)P2P_TPB_HOST * ptm;
            sl += rows * (double)((v[i + 3] - v[i + 2] + 31) / 32 * 32);
          }
        return sl;
      };
      double slots4 = 0.0;
      bool short_grid = false;   // fewer than ~10 waves of 512-point items: the tail dominates
      for (int c = force == 8 ? 0 : 1; c < 3; ++c) {
        if ((force == 3 || force == 4 || force == 8) && cand[c] != force) continue;
        p->p2p_pt = cand[c];
        tile = (int64_t)P2P_TPB_HOST * cand[c];
        build_items();
        const int64_t nit = (int64_t)(it[0].size() + it[1].size() + it[2].size()) / 4;
        if (cand[c] == force) break;
        if (cand[c] == 4) {
          slots4 = padded_slots(4);
          short_grid = nit < 10 * ctas[c] * (int64_t)nsm;
          if (!short_grid) {
            // enough waves: keep 512-point tiles unless the leaves fill them poorly -- 384-point
            // tiles must save > 8% of the padded slots to beat their lower per-slot rate (C4's
            // 3,676-point leaves: 6.7% fewer slots, measured 1% slower at 384; C5 at eps/10
            // (~305-point leaves): 512-point tiles are 60% full, 384-point tiles 79%)
            tile = (int64_t)P2P_TPB_HOST * 3;
            build_items();
            if (padded_slots(3) * 1.08 < slots4) {
              p->p2p_pt = 3;
              break;
            }
            tile = (int64_t)P2P_TPB_HOST * 4;
            build_items();
            break;
          }
        }
      }
      // Mixed tiles (default when the plan kept 512-point tiles; HFMM_P2P_MIX=0 opts out): each leaf is
      // cut into full 512-point tiles plus <= 384-point tiles, launched as two item classes (4 and 3
      // targets per thread), instead of a last 512-slot tile that is mostly padding.
      {
        const char *e = getenv("HFMM_P2P_MIX");
        const int mode = e ? atoi(e) : 1;   // 2: also on short grids (tests)
        if (!force && ((mode == 1 && p->p2p_pt == 4 && !short_grid) || mode == 2)) {
          p->p2p_pt = 4;
          mix_tiles = true;
          tile = (int64_t)P2P_TPB_HOST * 4;
          build_items();
          p->p2p_mix = true;
        }
      }
    // Row skipping (p2p_sym_kernel<..., RS = true>): warps skip their target rows wholly past the
    // tile's end.  Its per-slot rate is lower (same-box A/Bs, profiles/r02/rowskip_ab*.txt: C4 / C5
    // 0.7% / 2.4% slower with 5% / 4% dead slots; C3_acc 7% and C5_acc 4% faster with 29% / 17%
    // dead; C3, a short grid, 4% faster with 3.5%), so the plan turns it on when more than
    // HFMM_P2P_ROWSKIP_MIN (default 8%) of the tile slots are dead, or for short grids.
    {
      double thr = 0.08;
      if (const char *e = getenv("HFMM_P2P_ROWSKIP_MIN")) thr = atof(e);
      const double full = padded_slots(p->p2p_pt), live = padded_slots(p->p2p_pt, true);
      p->p2p_rowskip = !p->p2p_mix && p->p2p_pt != 8 && full > 0.0 &&
                       (live < (1.0 - thr) * full || (short_grid && thr < 1.0));
      p->p2p_dead_frac = full > 0.0 ? 1.0 - live / full : 0.0;
    }
    }
    // longest items first (LPT order against the tail of the grid)
    std::vector<int64_t> sorted_items[3];
    for (int k = 0; k < 3; ++k) {
      const int64_t m = (int64_t)it[k].size() / 4;
      std::vector<int64_t> ord(m);
      std::iota(ord.begin(), ord.end(), 0);
      auto cost = [&](int64_t i) { return (it[k][4 * i + 1] - it[k][4 * i]) * (it[k][4 * i + 3] - it[k][4 * i + 2]); };
      // mixed tiles: the 512-point class first (one launch per class), longest first inside a class
      auto small = [&](int64_t i) { return p->p2p_mix && it[k][4 * i + 1] - it[k][4 * i] <= 3 * (int64_t)P2P_TPB_HOST; };
      // run time of an item: every thread of the tile evaluates its PT targets, live or not (with
      // row skipping: its live 128-target rows), so a launch's items are ordered by their source
      // count (x live rows) -- a partly filled last tile runs as long as a full one
      // (HFMM_P2P_SORT=0: by live pairs)
      const bool by_slots = !(getenv("HFMM_P2P_SORT") && atoi(getenv("HFMM_P2P_SORT")) == 0);
      auto key = [&](int64_t i) {
        if (!by_slots || k == P2P_DIAG) return cost(i);
        const int64_t ns = it[k][4 * i + 3] - it[k][4 * i + 2];
        // row skipping: the item runs for the live 128-target rows of its first warp
        if (p->p2p_rowskip) return (it[k][4 * i + 1] - it[k][4 * i] + P2P_TPB_HOST - 1) / P2P_TPB_HOST * ns;
        return ns;
      };
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) {
        if (small(x) != small(y)) return small(y);
        return key(x) > key(y);
      });
      p->p2p_n4[k] = m;
      if (p->p2p_mix) {
        p->p2p_n4[k] = 0;
        for (int64_t i = 0; i < m; ++i) p->p2p_n4[k] += small(i) ? 0 : 1;
      }
      std::vector<int64_t> sorted(4 * m);
      for (int64_t i = 0; i < m; ++i)
        for (int c = 0; c < 4; ++c) sorted[4 * i + c] = it[k][4 * ord[i] + c];
      if (k == P2P_SYM)
        for (int64_t i = 0; i < m; ++i) sym_pairs += cost(i);
      if (k == P2P_DIAG && HFMM_P2P_DSYM)  // diagonal tiles: n (n - 1) / 2 unordered pairs each
        for (int64_t i = 0; i < m; ++i) {
          const int64_t nt = it[k][4 * i + 1] - it[k][4 * i];
          sym_pairs += nt * (nt - 1) / 2;
        }
      p->p2p_items[k] = dupload(sorted);
      sorted_items[k] = std::move(sorted);
      p->p2p_nitems[k] = m;
    }
    // deterministic accumulation (default; HFMM_ATOMIC_NEAR opts out): every item writes its row (and, for the
    // symmetric kernels, column) partial sums into its own slots; point i then sums its partials
    // in a fixed order (kinds in launch order, items in launch order, rows before columns)
    if (!(flags & HFMM_ATOMIC_NEAR)) {   // default (HFMM_DETERMINISTIC); +0.2% on C4, bitwise repeatable
      std::vector<int64_t> slot[3];
      int64_t off = 0;
      for (int k : {P2P_SYM, P2P_DIAG, P2P_ORD}) {
        const bool cols = k == P2P_SYM || (k == P2P_DIAG && HFMM_P2P_DSYM);
        const std::vector<int64_t> &v = sorted_items[k];
        const int64_t m = (int64_t)v.size() / 4;
        slot[k].assign(2 * m, -1);
        for (int64_t i = 0; i < m; ++i) {
          slot[k][2 * i] = off, off += v[4 * i + 1] - v[4 * i];
          if (cols) slot[k][2 * i + 1] = off, off += v[4 * i + 3] - v[4 * i + 2];
        }
      }
      std::vector<int64_t> rp(t.n + 1, 0), idx((size_t)off);
      for (int pass = 0; pass < 2; ++pass) {   // count, then fill
        std::vector<int64_t> fill;
        if (pass == 1) {
          for (int64_t i = 0; i < t.n; ++i) rp[i + 1] += rp[i];
          fill.assign(rp.begin(), rp.end() - 1);
        }
        for (int k : {P2P_SYM, P2P_DIAG, P2P_ORD}) {
          const std::vector<int64_t> &v = sorted_items[k];
          const int64_t m = (int64_t)v.size() / 4;
          for (int64_t i = 0; i < m; ++i) {
            for (int64_t q = v[4 * i]; q < v[4 * i + 1]; ++q) {
              if (pass == 0) ++rp[q + 1];
              else idx[(size_t)fill[q]++] = slot[k][2 * i] + (q - v[4 * i]);
            }
            if (slot[k][2 * i + 1] >= 0)
              for (int64_t q = v[4 * i + 2]; q < v[4 * i + 3]; ++q) {
                if (pass == 0) ++rp[q + 1];
                else idx[(size_t)fill[q]++] = slot[k][2 * i + 1] + (q - v[4 * i + 2]);
              }
          }
        }
      }
      for (int k = 0; k < 3; ++k) p->p2p_slot[k] = dupload(slot[k]);
      p->p2p_part = dalloc<double2>((size_t)std::max<int64_t>(off, 1));
      p->p2p_rp = dupload(rp);
      p->p2p_idx = dupload(idx);
      if (!p->p2p_part || !p->p2p_rp || (off && !p->p2p_idx)) {
        p->err = "hfmm_precompute: allocation failed (deterministic P2P partials)";
        return HFMM_E_NOMEM;
      }
    }
    // hfmm_direct: every target tile against all points (self pair masked)
    {
      std::vector<int64_t> d;
      for (int64_t t0 = 0; t0 < t.n; t0 += tile) d.insert(d.end(), {t0, std::min(t0 + tile, t.n), 0, t.n});
      p->dir_items = dupload(d);
      p->dir_nitems = (int64_t)d.size() / 4;
    }
    // source level: box point ranges; L2T tiles (kTile targets of one owned source box) unless
    // the boxes are small (< 64 points on average: warp-per-box S2M / L2T kernels)
    std::vector<int32_t> tl;
    std::vector<int64_t> tb;
    p->small_src = false;
    if (p->L_f >= 2) {
      const LevelBoxes &Bs = t.levels[p->D_s];
      const LevelDev &Ls = p->lv[p->D_s];
      const int64_t nown = Ls.own1 - Ls.own0;
      p->small_src = nown > 0 && (double)(Bs.first[Ls.own1] - Bs.first[Ls.own0]) < 64.0 * (double)nown;
      if (!p->small_src)
        for (int64_t b = Ls.own0; b < Ls.own1; ++b)
          for (int64_t s0 = Bs.first[b]; s0 < Bs.first[b + 1]; s0 += kTile) tl.push_back((int32_t)b), tb.push_back(s0);
      p->first_src = dupload(Bs.first);
    }
    p->first_near = dupload(B.first);
    p->tile_leaf = dupload(tl), p->tile_begin = dupload(tb);
    p->ntiles = (int64_t)tl.size();
    p->info.p2p_pairs = pairs;
    p->info.p2p_sym_pairs = sym_pairs;
    p->p2p_sym_pairs = sym_pairs;
    for (int d = 0; d < 3; ++d) {
      p->dummy_t[d] = (t.lo[d] - 3.0 * t.size) * p->uscale;
      p->dummy_s[d] = (t.lo[d] + 4.0 * t.size) * p->uscale;
    }
  }
  if (p->L_f >= 2) p->y_far = dalloc<double2>(t.n);
  CK(cudaStreamSynchronize(p->stream));
  CK(cudaGetLastError());
  // info
  hfmm_info &in = p->info;
  in.n = t.n, in.depth = D, in.L_f = p->L_f, in.kappa = kappa, in.eps = eps, in.alpha = alpha,
  in.tau = p->tau, in.rank = p->rank, in.nranks = p->nranks;
  in.nlevels = 0;
  for (int l = 2; l <= D && in.nlevels < HFMM_MAX_LEVELS; ++l) {
    const LevelDev &L = p->lv[l];
    hfmm_level_info &li = in.level[in.nlevels++];
    li.level = l, li.a = L.a, li.ell = L.ell, li.n_theta = L.nth, li.n_phi = L.nph, li.alpha = L.alpha, li.K = L.K,
    li.F = L.F, li.active = L.active ? 1 : 0, li.boxes = L.nbox, li.m2l_pairs = L.il_nnz;
    li.rep = L.rep ? 1 : 0;
    li.ragged = L.ragged ? 1 : 0;
    li.m2l_block = (L.m2lg && m2l_group_plan_kind(L.m2lg) == 1) ? 1 : 0;
    li.halo = L.halo ? 1 : 0;
    li.m_recv_boxes = li.m_send_boxes = 0;
    if (L.active && p->nranks > 1) {
      if (L.halo) {
        li.m_recv_boxes = L.hr_off.back(), li.m_send_boxes = L.hs_off.back();
      } else {
        li.m_recv_boxes = L.nbox - (L.own1 - L.own0);
        li.m_send_boxes = (L.own1 - L.own0) * (p->nranks - 1);
      }
    }
  }
  in.s2m_evals = p->L_f >= 2 ? (p->own_pt1 - p->own_pt0) * p->lv[p->D_s].K : 0;
  in.source_level = p->D_s;
  {  // kernel launches of one matvec (run_matvec): permute, P2P kinds, far chain, combine
    int nl = 2 + ((flags & HFMM_ATOMIC_NEAR) ? 0 : 1), n4 = 0;   // + the partial-sum reduction
    for (int k = 0; k < 3; ++k) {   // one launch per kind and (mixed tiles) tile class
      const int64_t c4 = p->p2p_mix ? p->p2p_n4[k] : p->p2p_nitems[k];
      nl += (c4 > 0 ? 1 : 0) + (p->p2p_nitems[k] > c4 ? 1 : 0);
    }
    if (p->L_f >= 2) {
      for (int l = p->D_s; l > 2; --l) {          // M2M: rows + cols pass per level (or one pass)
        const LevelDev &C = p->lv[l], &P = p->lv[l - 1];
        const bool sym = !C.ragged && !P.ragged && sym2_up_applies(C.nth, C.nph, P.nth, P.nph);
        n4 += sym ? 1 : 0;
        nl += (sym || (!C.ragged && !P.ragged && box2_up_applies(C.nth, C.nph, P.nth, P.nph))) ? 1 : 2;
      }
      for (int l = 2; l < p->D_s; ++l) {          // L2L: cols + rows pass per level (or one pass)
        const LevelDev &P = p->lv[l], &C = p->lv[l + 1];
        const bool sym = !C.ragged && !P.ragged && sym2_down_applies(P.nth, P.nph, C.nth, C.nph);
        n4 += sym ? 1 : 0;
        nl += (sym || (!C.ragged && !P.ragged && box2_down_applies(P.nth, P.nph, C.nth, C.nph))) ? 1 : 2;
      }
      nl += 2 + (p->L_f - 1);                      // S2M, L2T, M2L per active level
    }
    in.launches = nl;
    in.p2p_tile = P2P_TPB_HOST * p->p2p_pt;
    in.p2p_rowskip = p->p2p_rowskip ? 1 : 0;
    in.p2p_dead_frac = p->p2p_dead_frac;
    in.p2p_mixed_items = 0;
    if (p->p2p_mix)
      for (int k = 0; k < 3; ++k) in.p2p_mixed_items += p->p2p_nitems[k] - p->p2p_n4[k];
    in.next4_passes = n4;
  }
  in.owned_points = p->own_pt1 - p->own_pt0;
  p->have_plan = true;
  if (p->L_f < 0) {
    p->err = "no admissible far-field level: matvec is the direct sum";
    return HFMM_W_NO_FARFIELD;
  }
  if (p->L_f < D) {
    p->err = "levels " + std::to_string(p->L_f + 1) + ".." + std::to_string(D) +
             " inadmissible (low-frequency breakdown), far-field leaf level L_f = " + std::to_string(p->L_f);
    return HFMM_W_BREAKDOWN;
  }
  return HFMM_OK;
}

// ---- the matvec ------------------------------------------------------------------------------
// NVTX range for the launches of one pass (scoped; visible to ncu --nvtx / nsys)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static int allgather_level(hfmm_plan *p, LevelDev &L, cudaStream_t s) {
  if (p->nranks <= 1) return HFMM_OK;
  NvtxRange nv("hfmm:allgather M_l");
  // all-gather of M_l over variable-size Morton ranges: one broadcast per root, grouped
  CKN(ncclGroupStart());
  ncclResult_t gr_ = ncclSuccess;
  for (int r = 0; r < p->nranks; ++r) {
    size_t cnt = (size_t)(L.rhi[r] - L.rlo[r]) * L.K * 2;
    if (!cnt) continue;
    double *buf = (double *)(L.M + L.rlo[r] * L.K);
    CKG(ncclBroadcast(buf, buf, cnt, ncclDouble, r, p->comm, s));
  }
  CKN(ncclGroupEnd());
  return gr_ == ncclSuccess ? HFMM_OK : HFMM_E_NCCL;
}

// M2L halo of one level: grouped point-to-point sends of the packed owned boxes each peer needs and
// receives of the peers' boxes this rank needs, then one scatter into M_l
static int halo_level(hfmm_plan *p, LevelDev &L, cudaStream_t s) {
  if (p->nranks <= 1) return HFMM_OK;
  NvtxRange nv("hfmm:halo M_l");
  CKN(ncclGroupStart());
  ncclResult_t gr_ = ncclSuccess;
  for (int q = 0; q < p->nranks; ++q) {
    if (q == p->rank) continue;
    const size_t ns = (size_t)(L.hs_off[q + 1] - L.hs_off[q]) * L.K * 2, nr = (size_t)(L.hr_off[q + 1] - L.hr_off[q]) * L.K * 2;
    if (ns) CKG(ncclSend((const double *)(L.hs_buf + L.hs_off[q] * L.K), ns, ncclDouble, q, p->comm, s));
    if (nr) CKG(ncclRecv((double *)(L.hr_buf + L.hr_off[q] * L.K), nr, ncclDouble, q, p->comm, s));
  }
  CKN(ncclGroupEnd());
  if (gr_ != ncclSuccess) return HFMM_E_NCCL;
  if (L.hr_off.back() > 0) launch_gather_boxes(L.hr_buf, nullptr, L.M, L.hr_idx, L.hr_off.back(), L.K, s);
  return HFMM_OK;
}

// The matvec in two phases around its one exchange step (M2L needs the M_l of off-rank partners):
//   run_up    permute, near field (P2P, low-priority stream), S2M and M2M (far chain, high priority)
//   run_down  M2L, L2L, L2T on the far chain; join; combine
// run_matvec = run_up, all-gather of every active level's M (NCCL), run_down.  The virtual-rank
// group runs the phases of all its plans with peer copies in between.
static int run_up(hfmm_plan *p, const double2 *q_dev, cudaStream_t s_user, bool serial) {
  NvtxRange nv_up("hfmm:up (permute, P2P, S2M, M2M)");
  const Tree &t = p->tree;
  const int64_t n = t.n;
  const bool prof = p->profile;
  if (prof) cudaEventRecord(p->sev[0], s_user);
  launch_permute_q(q_dev, p->perm, p->q_sorted, n, s_user);
  PointsDev pts{p->px, p->py, p->pz, p->q_sorted};
  // near field (low priority) and far-field chain (high priority) forked from the caller's stream
  CK(cudaEventRecord(p->ev_fork, s_user));
  CK(cudaStreamWaitEvent(p->stream2, p->ev_fork, 0));
  cudaStream_t s = p->stream_hi;
  if (prof) cudaEventRecord(p->sev[7], p->stream2);
  const bool det = p->p2p_part != nullptr;
  if (!det) CK(cudaMemsetAsync(p->y_near, 0, n * sizeof(double2), p->stream2));
  {
    NvtxRange nv("hfmm:P2P");
    PointsU pu{p->ux, p->uy, p->uz, p->q_sorted};
    // mixed tiles: the <= 384-point class (3 targets per thread) on its own stream next to the
    // 512-point class when the partial sums go to per-item slots (det); behind it with atomics
    // (y_near is zeroed on stream2)
    const bool mix3 = p->p2p_mix && det && !serial;
    cudaStream_t s3 = mix3 ? p->stream3 : p->stream2;
    if (mix3) CK(cudaStreamWaitEvent(s3, p->ev_fork, 0));
    for (int k : {P2P_SYM, P2P_DIAG, P2P_ORD}) {
      const int kind = (k == P2P_DIAG && HFMM_P2P_DSYM) ? P2P_DSYM : k;
      const int64_t n4 = p->p2p_mix ? p->p2p_n4[k] : p->p2p_nitems[k];
      launch_p2p_items(pu, p->p2p_items[k], n4, kind, p->uscale, p->dummy_t, p->dummy_s, p->y_near, p->stream2,
                       p->p2p_pt, det ? p->p2p_part : nullptr, det ? p->p2p_slot[k] : nullptr, p->p2p_rowskip);
      if (p->p2p_nitems[k] > n4)
        launch_p2p_items(pu, p->p2p_items[k] + 4 * n4, p->p2p_nitems[k] - n4, kind, p->uscale, p->dummy_t,
                         p->dummy_s, p->y_near, s3, 3, det ? p->p2p_part : nullptr,
                         det ? p->p2p_slot[k] + 2 * n4 : nullptr, false);
    }
    if (mix3) {
      CK(cudaEventRecord(p->ev_mix, s3));
      CK(cudaStreamWaitEvent(p->stream2, p->ev_mix, 0));
    }
    if (det) launch_p2p_reduce(p->p2p_part, p->p2p_rp, p->p2p_idx, n, p->y_near, p->stream2);
  }
  if (prof) cudaEventRecord(p->sev[8], p->stream2);
  CK(cudaEventRecord(p->ev_join, p->stream2));
  // HFMM_SERIAL: the far chain starts after the near field (measurement of undisturbed kernels)
  CK(cudaStreamWaitEvent(p->stream_hi, serial ? p->ev_join : p->ev_fork, 0));
  const TwiddleSet &tw = global_twiddles(p->device);
  if (p->L_f >= 2) {
    const int Lf = p->L_f, Ds = p->D_s;
    LevelDev &F = p->lv[Ds];
    if (p->small_src)
      launch_s2m_small(pts, p->first_src, F.cx, F.cy, F.cz, (int32_t)F.own0, (int32_t)F.own1, F.ks, F.K, F.M, s);
    else
      launch_s2m(pts, p->first_src, F.cx, F.cy, F.cz, (int32_t)F.own0, (int32_t)F.own1, F.ks, F.K, F.M, s);
    if (prof) cudaEventRecord(p->sev[1], s);
    for (int l = Ds; l > 2; --l) {  // M2M, through the translation-only levels too
      LevelDev &C = p->lv[l], &P = p->lv[l - 1];
      if (C.own1 > C.own0) {
        const int64_t nc = C.own1 - C.own0;
        const double2 *src = C.M + C.own0 * C.K;
        if (C.ragged) {  // 5-step step 1 on the ragged child rows -> rectangular child grid
          launch_rag2rect(src, C.K, C.nth, C.rows_d, C.off_d, C.nph, nullptr, nullptr, nullptr, nc, C.nph, p->scr1,
                          tw, s);
          src = p->scr1;
        }
        if (!C.ragged && !P.ragged &&
            (launch_fused_up(src, P.own1 - P.own0, C.nth, C.nph, P.nth, P.nph, P.cbeg + P.own0, C.own0, C.oct,
                             P.shift, P.M + P.own0 * P.K, p->tmp, p->tmp_elems, p->fu_cnt, tw, s) ||
             launch_box2_up(src, P.own1 - P.own0, C.nth, C.nph, P.nth, P.nph, P.cbeg + P.own0, C.own0, C.oct, P.shift,
                            P.M + P.own0 * P.K, tw, s)))
          continue;  // single pass: fused two-pass (large grids) or one CTA per item (small grids)
        launch_rows_up(src, nc, C.nth, C.nph, P.nph, p->tmp, tw, s);
        if (P.ragged) {  // per-child parent fields, then step 5 + shift + sum on the ragged parent grid
          launch_cols_up(p->tmp, C.nth, P.nph, P.nth, nullptr, 0, nullptr, nc, nullptr, p->scr2, tw, s);
          launch_rect2rag(p->scr2, P.nth, P.nph, P.cbeg + P.own0, C.own0, C.oct, P.shift, nullptr, P.rows_d,
                          P.off_d, P.K, P.own1 - P.own0, P.M + P.own0 * P.K, tw, s);
        } else {
          // parents own0..own1 have children C.own0.. (contiguous); child index relative to C.own0
          launch_cols_up(p->tmp, C.nth, P.nph, P.nth, P.cbeg + P.own0, C.own0, C.oct, P.own1 - P.own0, P.shift,
                         P.M + P.own0 * P.K, tw, s);
        }
      }
    }
  }
  // M2L halos: pack the owned boxes every peer needs (sorted lists) before the exchange
  for (int l = 2; l <= p->L_f; ++l) {
    const LevelDev &L = p->lv[l];
    if (L.halo && L.hs_off.back() > 0)
      launch_gather_boxes(L.M, L.hs_idx, L.hs_buf, nullptr, L.hs_off.back(), L.K, p->stream_hi);
  }
  CK(cudaEventRecord(p->ev_up, p->stream_hi));
  return HFMM_OK;
}

static int run_down(hfmm_plan *p, cudaStream_t s_user, bool sorted_out) {
  NvtxRange nv_down("hfmm:down (M2L, L2L, L2T, combine)");
  const Tree &t = p->tree;
  const int64_t n = t.n;
  const bool prof = p->profile;
  PointsDev pts{p->px, p->py, p->pz, p->q_sorted};
  cudaStream_t s = p->stream_hi;
  const TwiddleSet &tw = global_twiddles(p->device);
  if (p->L_f >= 2) {
    const int Lf = p->L_f, Ds = p->D_s;
    LevelDev &F = p->lv[Ds];
    if (prof) cudaEventRecord(p->sev[2], s);
    for (int l = 2; l <= Lf; ++l) {  // M2L
      NvtxRange nv("hfmm:M2L");
      LevelDev &L = p->lv[l];
      m2l_group_apply(L.m2lg, L.T, L.perm, L.M, L.I, s);
    }
    if (prof) cudaEventRecord(p->sev[3], s);
    for (int l = 2; l < Ds; ++l) {  // L2L; L_2 = I_2; I = 0 below L_f (R-14)
      LevelDev &P = p->lv[l], &C = p->lv[l + 1];
      const double2 *Lp = (l == 2) ? P.I : P.L;
      if (C.own1 > C.own0) {
        const int64_t nc = C.own1 - C.own0;
        if (!P.ragged && !C.ragged &&
            launch_box2_down(Lp, nc, P.nth, P.nph, C.nth, C.nph, C.parent + C.own0, C.oct + C.own0, P.shift,
                             C.I ? C.I + C.own0 * C.K : nullptr, C.L + C.own0 * C.K, tw, s))
          continue;  // single pass (small square grids)
        if (P.ragged) {  // conj shift on the ragged parent grid + step 1 -> rectangular, per child
          launch_rag2rect(Lp, P.K, P.nth, P.rows_d, P.off_d, P.nph, C.parent + C.own0, C.oct + C.own0, P.shift, nc,
                          P.nph, p->scr2, tw, s);
          launch_cols_down(p->scr2, P.nth, P.nph, C.nth, nullptr, nullptr, nc, nullptr, p->tmp, tw, s);
        } else {
          launch_cols_down(Lp, P.nth, P.nph, C.nth, C.parent + C.own0, C.oct + C.own0, nc, P.shift, p->tmp, tw, s);
        }
        if (C.ragged) {  // rectangular child grid, then step 5 to the ragged rows + I_child
          launch_rows_down(p->tmp, nc, C.nth, P.nph, C.nph, nullptr, p->scr1, tw, s);
          launch_rect2rag(p->scr1, C.nth, C.nph, nullptr, 0, nullptr, nullptr, C.I ? C.I + C.own0 * C.K : nullptr,
                          C.rows_d, C.off_d, C.K, nc, C.L + C.own0 * C.K, tw, s);
        } else {
          launch_rows_down(p->tmp, nc, C.nth, P.nph, C.nph, C.I ? C.I + C.own0 * C.K : nullptr, C.L + C.own0 * C.K,
                           tw, s);
        }
      }
    }
    if (prof) cudaEventRecord(p->sev[4], s);
    const double2 *Lf_loc = (Ds == 2) ? F.I : F.L;
    const double wq = 8.0 * kPi * kPi / ((double)F.nth * (double)F.nph);
    if (p->small_src)
      launch_l2t_small(pts, p->first_src, F.cx, F.cy, F.cz, (int32_t)F.own0, (int32_t)F.own1, F.ks, F.K, Lf_loc, wq,
                       F.wk, p->y_far, s);
    else
      launch_l2t(pts, p->first_src, F.cx, F.cy, F.cz, p->tile_leaf, p->tile_begin, p->ntiles, F.ks, F.K, Lf_loc, wq,
                 F.wk, p->y_far, s);
    if (prof) cudaEventRecord(p->sev[5], s);
  } else if (prof) {
    for (int k = 1; k <= 5; ++k) cudaEventRecord(p->sev[k], s);
  }
  CK(cudaEventRecord(p->ev_join_hi, s));
  CK(cudaStreamWaitEvent(s_user, p->ev_join, 0));
  CK(cudaStreamWaitEvent(s_user, p->ev_join_hi, 0));
  // owned rows: into y_out in input order, or (multi-rank gather) into y_sorted in sorted order
  if (sorted_out)
    launch_combine(p->y_near, p->L_f >= 2 ? p->y_far : nullptr, nullptr, p->y_sorted, n, p->own_pt0, p->own_pt1,
                   s_user);
  else
    launch_combine(p->y_near, p->L_f >= 2 ? p->y_far : nullptr, p->perm, p->y_out, n, p->own_pt0, p->own_pt1,
                   s_user);
  if (prof) cudaEventRecord(p->sev[6], s_user);
  CK(cudaGetLastError());
  return HFMM_OK;
}

static int run_matvec(hfmm_plan *p, const double2 *q_dev, cudaStream_t s_user, bool serial, bool sorted_out) {
  int rc = run_up(p, q_dev, s_user, serial);
  if (rc) return rc;
  for (int l = 2; l <= p->L_f; ++l) {
    rc = p->lv[l].halo ? halo_level(p, p->lv[l], p->stream_hi) : allgather_level(p, p->lv[l], p->stream_hi);
    if (rc) return rc;
  }
  return run_down(p, s_user, sorted_out);
}

static int gather_y(hfmm_plan *p, cudaStream_t s) {
  if (p->nranks <= 1) return HFMM_OK;
  NvtxRange nv("hfmm:allgather y");
  // each rank wrote y of its owned sorted range [pt_lo[r], pt_hi[r]) into y_sorted: all-gather
  // of the (variable-size) ranges -- one broadcast per root, grouped -- then every rank
  // unpermutes the whole vector (N x 16 B per rank on the wire instead of an all-reduce's 2x)
  CKN(ncclGroupStart());
  ncclResult_t gr_ = ncclSuccess;
  for (int r = 0; r < p->nranks; ++r) {
    const size_t cnt = (size_t)(p->pt_hi[r] - p->pt_lo[r]) * 2;
    if (!cnt) continue;
    double *buf = (double *)(p->y_sorted + p->pt_lo[r]);
    CKG(ncclBroadcast(buf, buf, cnt, ncclDouble, r, p->comm, s));
  }
  CKN(ncclGroupEnd());
  if (gr_ != ncclSuccess) return HFMM_E_NCCL;
  launch_combine(p->y_sorted, nullptr, p->perm, p->y_out, p->tree.n, 0, p->tree.n, s);
  return HFMM_OK;
}

static int matvec_common(hfmm_plan *p, const double *q, double *y, int mem, void *stream, bool direct) {
  if (!p) return HFMM_E_ARG;
  if (!q || !y) {
    p->err = "matvec: NULL pointer";
    return HFMM_E_ARG;
  }
  if (!p->have_tree || (!direct && !p->have_plan)) {
    p->err = "matvec: build_tree and precompute first";
    return HFMM_E_STATE;
  }
  cudaSetDevice(p->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : p->stream;
  const int64_t n = p->tree.n;
  const bool host = (mem & 1) == HFMM_HOST;
  const bool local = (mem & HFMM_Y_LOCAL) != 0;
  const double2 *qd = (const double2 *)q;
  if (host) {
    CK(cudaMemcpyAsync(p->q_in, q, n * sizeof(double2), cudaMemcpyHostToDevice, s));
    qd = p->q_in;
  }
  if (p->vg && !direct) {
    p->err = "matvec: a virtual-rank plan runs through hfmm_vgroup_matvec";
    return HFMM_E_STATE;
  }
  const bool gather = p->nranks > 1 && !local && !direct;
  if (local || (p->nranks > 1 && direct)) CK(cudaMemsetAsync(p->y_out, 0, n * sizeof(double2), s));
  if (direct) {
    launch_permute_q(qd, p->perm, p->q_sorted, n, s);
    PointsU pu{p->ux, p->uy, p->uz, p->q_sorted};
    CK(cudaMemsetAsync(p->y_near, 0, n * sizeof(double2), s));
    launch_p2p_items(pu, p->dir_items, p->dir_nitems, P2P_DIAG, p->uscale, p->dummy_t, p->dummy_s, p->y_near, s,
                     p->p2p_pt);
    launch_combine(p->y_near, nullptr, p->perm, p->y_out, n, 0, n, s);
  } else {
    int rc = run_matvec(p, qd, s, (mem & HFMM_SERIAL) != 0, gather);
    if (rc) return rc;
    if (gather) {
      rc = gather_y(p, s);
      if (rc) return rc;
    }
  }
  if (host) {
    CK(cudaMemcpyAsync(y, p->y_out, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } else {
    CK(cudaMemcpyAsync(y, p->y_out, n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    if (!stream) CK(cudaStreamSynchronize(s));  // plan's own stream: complete before returning
  }
  if (p->profile && !direct) {
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, p->sev[0], p->sev[1]); p->stage_ms[0] = ms;
    cudaEventElapsedTime(&ms, p->sev[1], p->sev[2]); p->stage_ms[1] = ms;
    cudaEventElapsedTime(&ms, p->sev[2], p->sev[3]); p->stage_ms[2] = ms;
    cudaEventElapsedTime(&ms, p->sev[3], p->sev[4]); p->stage_ms[3] = ms;
    cudaEventElapsedTime(&ms, p->sev[4], p->sev[5]); p->stage_ms[4] = ms;
    cudaEventElapsedTime(&ms, p->sev[7], p->sev[8]); p->stage_ms[5] = ms;
    cudaEventElapsedTime(&ms, p->sev[0], p->sev[6]); p->stage_ms[6] = ms;
  }
  CK(cudaGetLastError());
  return HFMM_OK;
}

// ---- virtual ranks (test mode): R plans on one device, peer copies instead of NCCL ------------
extern "C" int hfmm_vgroup_create(hfmm_vgroup **out, int nranks) {
  if (!out || nranks < 1) return HFMM_E_ARG;
  *out = new hfmm_vgroup();
  (*out)->nranks = nranks;
  (*out)->plans.assign(nranks, nullptr);
  return HFMM_OK;
}

extern "C" void hfmm_vgroup_destroy(hfmm_vgroup *g) {
  if (!g) return;
  for (hfmm_plan *p : g->plans)
    if (p) p->vg = nullptr;
  delete g;
}

extern "C" int hfmm_set_dist_virtual(hfmm_plan *p, hfmm_vgroup *g, int rank) {
  if (!p) return HFMM_E_ARG;
  if (!g || rank < 0 || rank >= g->nranks || (g->plans[rank] && g->plans[rank] != p)) {
    p->err = "hfmm_set_dist_virtual: bad group / rank (or rank already taken)";
    return HFMM_E_ARG;
  }
  if (p->have_tree) {
    p->err = "hfmm_set_dist_virtual: must be called before build_tree";
    return HFMM_E_STATE;
  }
  if (p->comm) {
    ncclCommDestroy(p->comm);
    p->comm = nullptr;
  }
  p->rank = rank, p->nranks = g->nranks, p->vg = g;
  g->plans[rank] = p;
  return HFMM_OK;
}

extern "C" int hfmm_vgroup_matvec(hfmm_vgroup *g, const double *q, double *y, void *stream) {
  // The multi-rank matvec of run_matvec + gather_y with every collective replaced by one
  // cudaMemcpyAsync per peer block: (1) run_up on every rank; (2) for each active level, rank r
  // copies every peer r' 's owned block of M_l (after r' 's event) -- the all-gather; (3)
  // run_down on every rank (owned rows of y into its y_sorted); (4) rank r copies every peer's
  // owned range of y_sorted -- the y all-gather -- and unpermutes into y + r n.
  if (!g || !q || !y) return HFMM_E_ARG;
  const int R = g->nranks;
  for (hfmm_plan *p : g->plans)
    if (!p || !p->have_plan || p->device != g->plans[0]->device || p->tree.n != g->plans[0]->tree.n ||
        p->L_f != g->plans[0]->L_f)
      return HFMM_E_STATE;
  hfmm_plan *p0 = g->plans[0];
  cudaSetDevice(p0->device);
  cudaStream_t s = stream ? (cudaStream_t)stream : p0->stream;
  const int64_t n = p0->tree.n;
  for (hfmm_plan *p : g->plans) {
    int rc = run_up(p, (const double2 *)q, s, false);
    if (rc) return rc;
  }
  for (int r = 0; r < R; ++r) {
    hfmm_plan *p = g->plans[r];
    for (int rr = 0; rr < R; ++rr) {
      if (rr == r) continue;
      hfmm_plan *src = g->plans[rr];
      if (cudaStreamWaitEvent(p->stream_hi, src->ev_up, 0) != cudaSuccess) return HFMM_E_CUDA;
      for (int l = 2; l <= p->L_f; ++l) {
        LevelDev &L = p->lv[l], &S = src->lv[l];
        if (L.halo != S.halo) return HFMM_E_STATE;
        if (L.halo) {  // the peer's packed send segment for rank r -> rank r's receive segment from rr
          const int64_t cnt = L.hr_off[rr + 1] - L.hr_off[rr];
          if (cnt != S.hs_off[r + 1] - S.hs_off[r]) return HFMM_E_STATE;
          if (cnt > 0 &&
              cudaMemcpyAsync(L.hr_buf + L.hr_off[rr] * L.K, S.hs_buf + S.hs_off[r] * S.K,
                              (size_t)cnt * L.K * sizeof(double2), cudaMemcpyDeviceToDevice, p->stream_hi) != cudaSuccess)
            return HFMM_E_CUDA;
          continue;
        }
        const int64_t b0 = L.rlo[rr], b1 = L.rhi[rr];
        if (b1 > b0 &&
            cudaMemcpyAsync(L.M + b0 * L.K, S.M + b0 * S.K, (size_t)(b1 - b0) * L.K * sizeof(double2),
                            cudaMemcpyDeviceToDevice, p->stream_hi) != cudaSuccess)
          return HFMM_E_CUDA;
      }
    }
  }
  for (hfmm_plan *p : g->plans)  // scatter the received halos into M_l
    for (int l = 2; l <= p->L_f; ++l) {
      LevelDev &L = p->lv[l];
      if (L.halo && L.hr_off.back() > 0)
        launch_gather_boxes(L.hr_buf, nullptr, L.M, L.hr_idx, L.hr_off.back(), L.K, p->stream_hi);
    }
  for (hfmm_plan *p : g->plans) {
    int rc = run_down(p, s, true);
    if (rc) return rc;
  }
  for (int r = 0; r < R; ++r) {   // everything below is ordered on s after every run_down
    hfmm_plan *p = g->plans[r];
    for (int rr = 0; rr < R; ++rr) {
      const int64_t a = p->pt_lo[rr], b = p->pt_hi[rr];
      if (rr == r || b <= a) continue;
      if (cudaMemcpyAsync(p->y_sorted + a, g->plans[rr]->y_sorted + a, (size_t)(b - a) * sizeof(double2),
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return HFMM_E_CUDA;
    }
    launch_combine(p->y_sorted, nullptr, p->perm, (double2 *)y + (size_t)r * n, n, 0, n, s);
  }
  if (!stream && cudaStreamSynchronize(s) != cudaSuccess) return HFMM_E_CUDA;
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" int hfmm_matvec(hfmm_plan *p, const double *q, double *y, int mem, void *stream) {
  return matvec_common(p, q, y, mem, stream, false);
}

extern "C" int hfmm_direct(hfmm_plan *p, const double *q, double *y, int mem, void *stream) {
  if (p && !p->have_plan) {
    p->err = "hfmm_direct: call precompute first (kappa, scaled positions)";
    return HFMM_E_STATE;
  }
  return matvec_common(p, q, y, mem, stream, true);
}

extern "C" int hfmm_get_info(const hfmm_plan *p, hfmm_info *info) {
  if (!p || !info) return HFMM_E_ARG;
  if (!p->have_plan) return HFMM_E_STATE;
  *info = p->info;
  return HFMM_OK;
}

extern "C" int hfmm_stage_times(const hfmm_plan *p, double out[8]) {
  if (!p || !out) return HFMM_E_ARG;
  for (int i = 0; i < 8; ++i) out[i] = p->stage_ms[i];
  return HFMM_OK;
}

extern "C" int hfmm_debug_copy(const hfmm_plan *p, int what, int level, void *host_out, int64_t nbytes,
                               int64_t *needed) {
  if (!p) return HFMM_E_ARG;
  cudaSetDevice(p->device);
  const void *src = nullptr;
  int64_t bytes = 0;
  std::vector<int64_t> hostbuf;
  if (what >= 0 && what <= 3) {
    if (level < 2 || level >= (int)p->lv.size() || (what != 3 && level > std::max(p->L_f, p->D_s)))
      return HFMM_E_ARG;
    const LevelDev &L = p->lv[level];
    if (what == 3) {
      // the 316 tables T_o[k] = T_c(o)[perm_op(o)[k]], expanded from the 34 canonical ones
      bytes = (int64_t)316 * L.K * 16;
      if (needed) *needed = bytes;
      if (!host_out) return HFMM_OK;
      if (nbytes < bytes) return HFMM_E_ARG;
      if (!L.T || !L.perm) return HFMM_E_STATE;
      std::vector<int> cids, sym_of;
      canonical_offsets(cids, sym_of);
      std::vector<double2> T34((size_t)cids.size() * L.K);
      std::vector<int32_t> pm((size_t)16 * L.K);
      if (cudaMemcpy(T34.data(), L.T, T34.size() * 16, cudaMemcpyDeviceToHost) != cudaSuccess ||
          cudaMemcpy(pm.data(), L.perm, pm.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HFMM_E_CUDA;
      double2 *dst = (double2 *)host_out;
      for (int id = 0; id < 316; ++id) {
        const int c = sym_of[id] >> 4, op = sym_of[id] & 15;
        for (int64_t k = 0; k < L.K; ++k) dst[(size_t)id * L.K + k] = T34[(size_t)c * L.K + pm[(size_t)op * L.K + k]];
      }
      return HFMM_OK;
    } else {
      const double2 *b = what == 0 ? L.M : what == 1 ? L.I : (level == 2 ? L.I : L.L);
      src = b, bytes = L.nbox * L.K * 16;
    }
  } else if (what == 4) {
    src = p->y_near, bytes = p->tree.n * 16;
  } else if (what == 5) {
    src = p->y_far, bytes = p->y_far ? p->tree.n * 16 : 0;
  } else if (what == 6) {
    hostbuf = p->tree.perm;
  } else if (what == 7) {
    if (level < 0 || level > p->tree.depth) return HFMM_E_ARG;
    const LevelBoxes &B = p->tree.levels[level];
    for (int64_t b = 0; b < B.nbox(); ++b) {
      hostbuf.push_back(B.ix[b]), hostbuf.push_back(B.iy[b]), hostbuf.push_back(B.iz[b]);
      hostbuf.push_back(B.first[b]);
    }
  } else {
    return HFMM_E_ARG;
  }
  if (what >= 6) bytes = (int64_t)hostbuf.size() * 8;
  if (needed) *needed = bytes;
  if (!host_out) return HFMM_OK;
  if (nbytes < bytes) return HFMM_E_ARG;
  if (what >= 6) {
    std::memcpy(host_out, hostbuf.data(), bytes);
    return HFMM_OK;
  }
  if (!src || !bytes) return HFMM_E_STATE;
  if (cudaMemcpy(host_out, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return HFMM_E_CUDA;
  return HFMM_OK;
}

extern "C" const char *hfmm_last_error(const hfmm_plan *p) {
  return p ? p->err.c_str() : g_create_err.c_str();
}

extern "C" void hfmm_destroy(hfmm_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  free_levels(p);
  free_points(p);
  if (p->comm) ncclCommDestroy(p->comm);
  for (auto &e : p->sev)
    if (e) cudaEventDestroy(e);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_join) cudaEventDestroy(p->ev_join);
  if (p->ev_join_hi) cudaEventDestroy(p->ev_join_hi);
  if (p->ev_mix) cudaEventDestroy(p->ev_mix);
  if (p->stream3) cudaStreamDestroy(p->stream3);
  if (p->ev_up) cudaEventDestroy(p->ev_up);
  if (p->vg && p->rank < (int)p->vg->plans.size() && p->vg->plans[p->rank] == p) p->vg->plans[p->rank] = nullptr;
  if (p->stream_hi) cudaStreamDestroy(p->stream_hi);
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->stream2) cudaStreamDestroy(p->stream2);
  delete p;
}

// ---- operator entry points (BASELINE config 2 microbench) ------------------------------------
namespace {
struct OpCache {
  int32_t *cbeg = nullptr, *par = nullptr;
  int8_t *oct = nullptr;
  int64_t n = 0;
  void ensure(int64_t nparent) {
    if (nparent <= n) return;
    if (cbeg) cudaFree(cbeg), cudaFree(par), cudaFree(oct);
    std::vector<int32_t> cb(nparent + 1), pr(nparent * 8);
    std::vector<int8_t> oc(nparent * 8);
    for (int64_t i = 0; i <= nparent; ++i) cb[i] = (int32_t)(8 * i);
    for (int64_t c = 0; c < nparent * 8; ++c) pr[c] = (int32_t)(c / 8), oc[c] = (int8_t)(c % 8);
    cbeg = dupload(cb), par = dupload(pr), oct = dupload(oc);
    n = nparent;
  }
};
OpCache &op_cache() {  // per device: the index arrays live in that device's memory
  std::lock_guard<std::recursive_mutex> lk(cache_mutex());
  static std::map<int, OpCache> caches;
  int d = 0;
  cudaGetDevice(&d);
  return caches[d];
}
int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
bool up_or_down(int nth, int nph, int nth2, int nph2, bool *up) {
  if (nth2 >= nth && nph2 >= nph) *up = true;
  else if (nth2 <= nth && nph2 <= nph) *up = false;
  else return false;
  return (nth % 2 == 0) && (nth2 % 2 == 0) && (nph % 2 == 0) && (nph2 % 2 == 0) && seven_smooth(nth) &&
         seven_smooth(nth2) && seven_smooth(nph) && seven_smooth(nph2) && nth < kMaxFFT && nth2 < kMaxFFT &&
         nph < kMaxFFT && nph2 < kMaxFFT;
}
}  // namespace

extern "C" int64_t hfmm_resample_workspace(int nbatch, int n_theta, int n_phi, int n_theta2, int n_phi2) {
  bool up;
  if (!up_or_down(n_theta, n_phi, n_theta2, n_phi2, &up)) return -1;
  // UP: the rows-pass intermediate (or the fused kernel's ring) + its 2 nbatch + 1 task counters
  if (up) return (int64_t)nbatch * (n_theta / 2 + 1) * n_phi2 * 16 + ((int64_t)(2 * nbatch + 1) * 4 + 15) / 16 * 16;
  return (int64_t)nbatch * n_theta2 * (n_phi / 2) * 16;
}

extern "C" int hfmm_resample(int nbatch, int nth, int nph, int nth2, int nph2, const double *in, double *out,
                             void *work, void *stream) {
  bool up;
  if (nbatch < 0 || !in || !out || !up_or_down(nth, nph, nth2, nph2, &up)) return HFMM_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const TwiddleSet &tw = global_twiddles(cur_device());
  double2 *tmp = (double2 *)work;
  bool own = false;
  if (!tmp) {
    if (cudaMalloc(&tmp, hfmm_resample_workspace(nbatch, nth, nph, nth2, nph2)) != cudaSuccess) return HFMM_E_NOMEM;
    own = true;
  }
  if (up) {
    const size_t ring = (size_t)nbatch * (nth / 2 + 1) * nph2;   // complex values before the counters
    if (launch_fused_up((const double2 *)in, nbatch, nth, nph, nth2, nph2, nullptr, 0, nullptr, nullptr,
                        (double2 *)out, tmp, ring, (int *)(tmp + ring), tw, s)) {
    } else if (!launch_box2_up((const double2 *)in, nbatch, nth, nph, nth2, nph2, nullptr, 0, nullptr, nullptr,
                               (double2 *)out, tw, s)) {
      launch_rows_up((const double2 *)in, nbatch, nth, nph, nph2, tmp, tw, s);
      launch_cols_up(tmp, nth, nph2, nth2, nullptr, 0, nullptr, nbatch, nullptr, (double2 *)out, tw, s);
    }
  } else if (!launch_box2_down((const double2 *)in, nbatch, nth, nph, nth2, nph2, nullptr, nullptr, nullptr, nullptr,
                               (double2 *)out, tw, s)) {
    launch_cols_down((const double2 *)in, nth, nph, nth2, nullptr, nullptr, nbatch, nullptr, tmp, tw, s);
    launch_rows_down(tmp, nbatch, nth2, nph, nph2, nullptr, (double2 *)out, tw, s);
  }
  if (own) {
    cudaStreamSynchronize(s);
    cudaFree(tmp);
  }
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" int hfmm_m2m_op(int nparent, int nth, int nph, int nth2, int nph2, const double *child,
                           const double *shift, double *parent, void *work, void *stream) {
  bool up;
  if (nparent < 0 || !child || !parent || !up_or_down(nth, nph, nth2, nph2, &up) || !up) return HFMM_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const TwiddleSet &tw = global_twiddles(cur_device());
  OpCache &c = op_cache();
  {
    std::lock_guard<std::recursive_mutex> lk(cache_mutex());
    c.ensure(nparent);
  }
  double2 *tmp = (double2 *)work;
  bool own = false;
  if (!tmp) {
    if (cudaMalloc(&tmp, hfmm_resample_workspace(nparent * 8, nth, nph, nth2, nph2)) != cudaSuccess) return HFMM_E_NOMEM;
    own = true;
  }
  const size_t ring = (size_t)nparent * 8 * (nth / 2 + 1) * nph2;
  if (launch_fused_up((const double2 *)child, nparent, nth, nph, nth2, nph2, c.cbeg, 0, c.oct, (const double2 *)shift,
                      (double2 *)parent, tmp, ring, (int *)(tmp + ring), tw, s)) {
  } else if (!launch_box2_up((const double2 *)child, nparent, nth, nph, nth2, nph2, c.cbeg, 0, c.oct,
                             (const double2 *)shift, (double2 *)parent, tw, s)) {
    launch_rows_up((const double2 *)child, (int64_t)nparent * 8, nth, nph, nph2, tmp, tw, s);
    launch_cols_up(tmp, nth, nph2, nth2, c.cbeg, 0, c.oct, nparent, (const double2 *)shift, (double2 *)parent, tw, s);
  }
  if (own) {
    cudaStreamSynchronize(s);
    cudaFree(tmp);
  }
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" int hfmm_l2l_op(int nparent, int nth, int nph, int nth2, int nph2, const double *parent,
                           const double *shift, const double *incoming, double *child_out, void *work,
                           void *stream) {
  bool up;
  if (nparent < 0 || !parent || !child_out || !up_or_down(nth, nph, nth2, nph2, &up) || up) return HFMM_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const TwiddleSet &tw = global_twiddles(cur_device());
  OpCache &c = op_cache();
  {
    std::lock_guard<std::recursive_mutex> lk(cache_mutex());
    c.ensure(nparent);
  }
  double2 *tmp = (double2 *)work;
  bool own = false;
  if (!tmp) {
    if (cudaMalloc(&tmp, hfmm_resample_workspace(nparent * 8, nth, nph, nth2, nph2)) != cudaSuccess) return HFMM_E_NOMEM;
    own = true;
  }
  if (!launch_box2_down((const double2 *)parent, (int64_t)nparent * 8, nth, nph, nth2, nph2, c.par, c.oct,
                        (const double2 *)shift, (const double2 *)incoming, (double2 *)child_out, tw, s)) {
    launch_cols_down((const double2 *)parent, nth, nph, nth2, c.par, c.oct, (int64_t)nparent * 8,
                     (const double2 *)shift, tmp, tw, s);
    launch_rows_down(tmp, (int64_t)nparent * 8, nth2, nph, nph2, (const double2 *)incoming, (double2 *)child_out, tw, s);
  }
  if (own) {
    cudaStreamSynchronize(s);
    cudaFree(tmp);
  }
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" int hfmm_m2l_op_plan(int nbox, int64_t K, const int *row, const int *src, const int *oid, void **plan) {
  if (nbox < 0 || K <= 0 || !row || !src || !oid || !plan) return HFMM_E_ARG;
  for (int64_t e = 0; e < row[nbox]; ++e)
    if (oid[e] < 0 || oid[e] >= 316 || src[e] < 0 || src[e] >= nbox) return HFMM_E_ARG;
  *plan = m2l_group_plan_create(nbox, K, row, src, oid, nullptr);
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" int hfmm_m2l_op_apply(const void *plan, const double *T, const double *M, double *out, void *stream) {
  if (!plan || !T || !M || !out) return HFMM_E_ARG;
  m2l_group_apply((const M2LGroupPlan *)plan, (const double2 *)T, nullptr, (const double2 *)M, (double2 *)out,
                  (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? HFMM_OK : HFMM_E_CUDA;
}

extern "C" void hfmm_m2l_op_free(void *plan) { m2l_group_plan_destroy((M2LGroupPlan *)plan); }

extern "C" int hfmm_m2l_op_kind(const void *plan) { return m2l_group_plan_kind((const M2LGroupPlan *)plan); }

extern "C" int hfmm_m2l_op(int nbox, int64_t K, const int *row, const int *src, const int *oid, const double *T,
                           const double *M, double *out, void *stream) {
  if (nbox < 0 || K <= 0 || !row || !src || !oid || !T || !M || !out) return HFMM_E_ARG;
  // device CSR -> host, one-shot plan (hfmm_m2l_op_plan / _apply for repeated use)
  std::vector<int32_t> hr(nbox + 1);
  if (cudaMemcpy(hr.data(), row, hr.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) return HFMM_E_CUDA;
  std::vector<int32_t> hs(hr[nbox]), ho(hr[nbox]);
  if (cudaMemcpy(hs.data(), src, hs.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(ho.data(), oid, ho.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return HFMM_E_CUDA;
  void *pl = nullptr;
  int rc = hfmm_m2l_op_plan(nbox, K, hr.data(), hs.data(), ho.data(), &pl);
  if (rc) return rc;
  rc = hfmm_m2l_op_apply(pl, T, M, out, stream);
  cudaStreamSynchronize((cudaStream_t)stream);
  hfmm_m2l_op_free(pl);
  return rc;
}
