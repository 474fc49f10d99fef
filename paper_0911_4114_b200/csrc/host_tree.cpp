// Octree in Morton order (product code).
//   P:33   root level 0, a_l = a_0 / 2^l
//   P:114  boxes B^l_alpha with centres c^l_alpha; leaves own contiguous point ranges
// Points are sorted by the Morton key of their depth-D box (ties: input index), so every
// box of every level l <= D owns one contiguous range of the sorted arrays.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <map>
#include <string>
#include <tuple>

#include "hfmm_impl.h"
#include "../../include/hfmm.h"

namespace hfmm {

static inline uint32_t spread3(uint32_t v) {  // 10 bits -> every third bit
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

uint32_t morton3(uint32_t x, uint32_t y, uint32_t z) {
  return (spread3(x) << 2) | (spread3(y) << 1) | spread3(z);
}

int32_t LevelBoxes::find(int x, int y, int z) const {
  const int n = 1 << level;
  if (x < 0 || y < 0 || z < 0 || x >= n || y >= n || z >= n) return -1;
  uint32_t k = morton3((uint32_t)x, (uint32_t)y, (uint32_t)z);
  auto it = std::lower_bound(key.begin(), key.end(), k);
  if (it == key.end() || *it != k) return -1;
  return (int32_t)(it - key.begin());
}

int offset_id(int ox, int oy, int oz) {
  // lexicographic enumeration of [-3,3]^3 minus [-1,1]^3
  int id = 0;
  for (int x = -3; x <= 3; ++x)
    for (int y = -3; y <= 3; ++y)
      for (int z = -3; z <= 3; ++z) {
        if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) < 2) continue;
        if (x == ox && y == oy && z == oz) return id;
        ++id;
      }
  return -1;
}

void offset_vec(int id, int o[3]) {
  int k = 0;
  for (int x = -3; x <= 3; ++x)
    for (int y = -3; y <= 3; ++y)
      for (int z = -3; z <= 3; ++z) {
        if (std::max(std::abs(x), std::max(std::abs(y), std::abs(z))) < 2) continue;
        if (k == id) {
          o[0] = x, o[1] = y, o[2] = z;
          return;
        }
        ++k;
      }
}

int build_tree(const double *xyz, int64_t n, int depth, const double lo[3], double size, Tree &t,
               std::string &err) {
  if (n <= 0 || depth < 2 || depth > 10 || !(size > 0) || !std::isfinite(size)) {
    err = "build_tree: need n > 0, 2 <= depth <= 10, finite size > 0";
    return HFMM_E_ARG;
  }
  for (int d = 0; d < 3; ++d)
    if (!std::isfinite(lo[d])) {
      err = "build_tree: non-finite root corner";
      return HFMM_E_ARG;
    }
  t = Tree();
  t.n = n;
  t.depth = depth;
  t.size = size;
  for (int d = 0; d < 3; ++d) t.lo[d] = lo[d];
  const int nb = 1 << depth;
  const double a = size / nb;
  std::vector<uint32_t> key(n);
  for (int64_t i = 0; i < n; ++i) {
    int b[3];
    for (int d = 0; d < 3; ++d) {
      double v = xyz[3 * i + d];
      if (!std::isfinite(v)) {
        err = "build_tree: non-finite coordinate at point " + std::to_string(i);
        return HFMM_E_ARG;
      }
      double u = std::floor((v - lo[d]) / a);
      if (u < 0 || v > lo[d] + size) {
        err = "build_tree: point " + std::to_string(i) + " outside the root cube";
        return HFMM_E_DOMAIN;
      }
      b[d] = std::min((int)u, nb - 1);
    }
    key[i] = morton3(b[0], b[1], b[2]);
  }
  t.perm.resize(n);
  std::iota(t.perm.begin(), t.perm.end(), 0);
  std::stable_sort(t.perm.begin(), t.perm.end(), [&](int64_t u, int64_t v) { return key[u] < key[v]; });
  t.xs.resize(n), t.ys.resize(n), t.zs.resize(n);
  std::vector<uint32_t> skey(n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = t.perm[i];
    t.xs[i] = xyz[3 * j], t.ys[i] = xyz[3 * j + 1], t.zs[i] = xyz[3 * j + 2];
    skey[i] = key[j];
  }
  // exact duplicates (kernel undefined): identical points share a leaf key
  {
    int64_t i = 0;
    while (i < n) {
      int64_t e = i;
      while (e < n && skey[e] == skey[i]) ++e;
      if (e - i > 1) {
        std::vector<int64_t> idx(e - i);
        std::iota(idx.begin(), idx.end(), i);
        std::sort(idx.begin(), idx.end(), [&](int64_t u, int64_t v) {
          if (t.xs[u] != t.xs[v]) return t.xs[u] < t.xs[v];
          if (t.ys[u] != t.ys[v]) return t.ys[u] < t.ys[v];
          return t.zs[u] < t.zs[v];
        });
        for (size_t k = 1; k < idx.size(); ++k) {
          int64_t u = idx[k - 1], v = idx[k];
          if (t.xs[u] == t.xs[v] && t.ys[u] == t.ys[v] && t.zs[u] == t.zs[v]) {
            err = "build_tree: coincident points (input " + std::to_string(t.perm[u]) + ", " +
                  std::to_string(t.perm[v]) + ")";
            return HFMM_E_COINCIDENT;
          }
        }
      }
      i = e;
    }
  }
  t.levels.resize(depth + 1);
  for (int l = 0; l <= depth; ++l) {
    LevelBoxes &L = t.levels[l];
    L.level = l;
    L.a = size / (double)(1 << l);
    const int shift = 3 * (depth - l);
    int64_t i = 0;
    while (i < n) {
      uint32_t k = skey[i] >> shift;
      L.key.push_back(k);
      L.first.push_back(i);
      while (i < n && (skey[i] >> shift) == k) ++i;
    }
    L.first.push_back(n);
    for (uint32_t k : L.key) {
      uint32_t x = 0, y = 0, z = 0;
      for (int b = 0; b < l; ++b) {
        x |= ((k >> (3 * b + 2)) & 1u) << b;
        y |= ((k >> (3 * b + 1)) & 1u) << b;
        z |= ((k >> (3 * b + 0)) & 1u) << b;
      }
      L.ix.push_back(x), L.iy.push_back(y), L.iz.push_back(z);
    }
  }
  for (int l = 1; l <= depth; ++l) {
    LevelBoxes &L = t.levels[l];
    const LevelBoxes &P = t.levels[l - 1];
    L.parent.resize(L.nbox());
    for (int64_t b = 0; b < L.nbox(); ++b) L.parent[b] = P.find(L.ix[b] >> 1, L.iy[b] >> 1, L.iz[b] >> 1);
  }
  for (int l = 0; l < depth; ++l) {
    LevelBoxes &L = t.levels[l];
    const LevelBoxes &C = t.levels[l + 1];
    L.child_begin.assign(L.nbox() + 1, 0);
    for (int64_t c = 0; c < C.nbox(); ++c) L.child_begin[C.parent[c] + 1]++;
    for (int64_t b = 0; b < L.nbox(); ++b) L.child_begin[b + 1] += L.child_begin[b];
  }
  return 0;
}

// Multi-GPU ownership: contiguous Morton ranges of level-2 boxes (whole subtrees) for R ranks,
// balanced by an estimate of FP64 work per level-2 subtree: P2P pairs of its leaves at L_f plus
// 2 n_leaf K (S2M + L2T evaluations).  cut[r]..cut[r+1] is rank r's range.
void partition_level2(const Tree &t, int L_f, int64_t K, int R, std::vector<int64_t> &cut) {
  const LevelBoxes &B2 = t.levels[2];
  const LevelBoxes &BL = t.levels[L_f];
  std::vector<double> w(B2.nbox(), 0.0);
  for (int64_t b = 0; b < BL.nbox(); ++b) {
    int64_t nb = BL.first[b + 1] - BL.first[b];
    int64_t src = 0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          int32_t k = BL.find(BL.ix[b] + dx, BL.iy[b] + dy, BL.iz[b] + dz);
          if (k >= 0) src += BL.first[k + 1] - BL.first[k];
        }
    int32_t a = (int32_t)b;
    for (int l = L_f; l > 2; --l) a = t.levels[l].parent[a];
    w[a] += (double)nb * (double)src + 2.0 * (double)nb * (double)K;
  }
  double tot = 0.0;
  for (double v : w) tot += v;
  cut.assign(R + 1, B2.nbox());
  cut[0] = 0;
  double acc = 0;
  int k = 1;
  for (int64_t b = 0; b < B2.nbox() && k < R; ++b) {
    acc += w[b];
    while (k < R && acc >= tot * k / R) cut[k++] = b + 1;
  }
  for (; k < R; ++k) cut[k] = B2.nbox();
}

// M2L halo lists of rank r at level l (multi-rank plans; used by hfmm_precompute and exported as
// hfmm_halo_lists): recv[q] = the boxes owned by q != r in the interaction list (children of
// the parent's neighbours that are not adjacent) of a box owned by r; send[q] = the boxes owned by r
// in the interaction list of a box owned by q.  Sorted and unique, so the sender's send[r'] and the
// receiver's recv[r] are the same list.  rlo / rhi: every rank's owned box range at level l.
void m2l_halo_lists(const Tree &t, int l, const std::vector<int64_t> &rlo, const std::vector<int64_t> &rhi, int r,
                    std::vector<std::vector<int64_t>> &snd, std::vector<std::vector<int64_t>> &rcv) {
  const LevelBoxes &B = t.levels[l];
  const int R = (int)rlo.size();
  snd.assign(R, {}), rcv.assign(R, {});
  auto owner = [&](int64_t b) {
    for (int q = 0; q < R; ++q)
      if (b >= rlo[q] && b < rhi[q]) return q;
    return -1;
  };
  for (int64_t b = 0; b < B.nbox(); ++b) {
    const int ob = owner(b);
    if (ob < 0) continue;
    const int px = B.ix[b] >> 1, py = B.iy[b] >> 1, pz = B.iz[b] >> 1;
    for (int dx = -3; dx <= 3; ++dx)
      for (int dy = -3; dy <= 3; ++dy)
        for (int dz = -3; dz <= 3; ++dz) {
          if (std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz))) < 2) continue;
          const int x = B.ix[b] + dx, y = B.iy[b] + dy, z = B.iz[b] + dz;
          if (std::abs((x >> 1) - px) > 1 || std::abs((y >> 1) - py) > 1 || std::abs((z >> 1) - pz) > 1) continue;
          const int32_t k = B.find(x, y, z);
          if (k < 0) continue;
          const int os = owner(k);
          if (os < 0 || os == ob) continue;
          if (ob == r) rcv[os].push_back(k);
          else if (os == r) snd[ob].push_back(k);
        }
  }
  for (int q = 0; q < R; ++q)
    for (auto *v : {&snd[q], &rcv[q]}) {
      std::sort(v->begin(), v->end());
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
}

// 34 canonical transfer vectors (Fig. SemiOctant): x >= y >= 0, z >= 0, in the
// lexicographic order of the 316.  Offset o = F P c with c canonical, P the x<->y swap (when
// |o_y| > |o_x|) and F the sign flips of o's negative components, so
//   T_o(s) = T_c((F P)^T s) = T_c(P F s)
// and on the quadrature (N_theta even, N_phi = 0 mod 4) every reflection maps grid points to grid
// points: z-flip theta -> pi - theta (n -> N_theta/2 - n), x-flip phi -> pi - phi (m -> N_phi/2 - m),
// y-flip phi -> -phi, swap phi -> pi/2 - phi (m -> N_phi/4 - m), folded back into the stored half
// with eqn:NumSphereSym.  op = fx | fy << 1 | fz << 2 | swap << 3.
void canonical_offsets(std::vector<int> &cids, std::vector<int> &sym_of /*[316]: cid << 4 | op*/) {
  cids.clear();
  std::map<std::tuple<int, int, int>, int> cidx;
  for (int id = 0; id < 316; ++id) {
    int o[3];
    offset_vec(id, o);
    if (o[0] >= o[1] && o[1] >= 0 && o[2] >= 0) {
      cidx[std::make_tuple(o[0], o[1], o[2])] = (int)cids.size();
      cids.push_back(id);
    }
  }
  sym_of.assign(316, 0);
  for (int id = 0; id < 316; ++id) {
    int o[3];
    offset_vec(id, o);
    const int ax = std::abs(o[0]), ay = std::abs(o[1]), az = std::abs(o[2]);
    const int sw = ay > ax ? 1 : 0;
    const int c = cidx.at(std::make_tuple(std::max(ax, ay), std::min(ax, ay), az));
    const int op = (o[0] < 0 ? 1 : 0) | (o[1] < 0 ? 2 : 0) | (o[2] < 0 ? 4 : 0) | (sw << 3);
    sym_of[id] = (c << 4) | op;
  }
}

// perm[op][k]: stored index of the canonical table holding T_o at stored point k
void symmetry_perms(int nth, int nph, std::vector<int32_t> &perm) {
  const int h = nph / 2;
  const int64_t K = (int64_t)nth * h;
  perm.assign((size_t)16 * K, 0);
  for (int op = 0; op < 16; ++op)
    for (int n = 0; n < nth; ++n)
      for (int m = 0; m < h; ++m) {
        int nn = n, mm = m;  // full-torus indices, 0 <= mm < nph
        if (op & 1) mm = (nph / 2 - mm + nph) % nph;      // x -> -x: phi -> pi - phi
        if (op & 2) mm = (nph - mm) % nph;                // y -> -y: phi -> -phi
        if (op & 4) nn = (nth / 2 - nn + nth) % nth;      // z -> -z: theta -> pi - theta
        if (op & 8) mm = ((nph / 4 - mm) % nph + nph) % nph;  // x <-> y: phi -> pi/2 - phi
        if (mm >= h) nn = (nth - nn) % nth, mm -= h;      // eqn:NumSphereSym
        perm[(size_t)op * K + (int64_t)n * h + m] = (int32_t)((int64_t)nn * h + mm);
      }
}


}  // namespace hfmm

extern "C" int hfmm_partition(int64_t n, const double *xyz, int depth, const double lo[3], double size,
                              int L_f, int64_t K, int nranks, int64_t *cuts, int64_t *pt_ranges,
                              int64_t *perm) {
  using namespace hfmm;
  if (!xyz || !lo || !cuts || !pt_ranges || nranks < 1 || L_f < 2 || L_f > depth || K <= 0)
    return HFMM_E_ARG;
  Tree t;
  std::string err;
  int rc = build_tree(xyz, n, depth, lo, size, t, err);
  if (rc) return rc;
  std::vector<int64_t> cut;
  partition_level2(t, L_f, K, nranks, cut);
  for (int r = 0; r <= nranks; ++r) cuts[r] = cut[r];
  for (int r = 0; r < nranks; ++r) {
    int64_t b0 = cut[r], b1 = cut[r + 1];
    for (int l = 2; l < L_f; ++l) {  // descend to L_f (children ranges are contiguous)
      b0 = t.levels[l].child_begin[b0];
      b1 = t.levels[l].child_begin[b1];
    }
    pt_ranges[2 * r] = t.levels[L_f].first[b0];
    pt_ranges[2 * r + 1] = t.levels[L_f].first[b1];
  }
  if (perm)
    for (int64_t i = 0; i < n; ++i) perm[i] = t.perm[i];
  return 0;
}

extern "C" int hfmm_halo_lists(int64_t n, const double *xyz, int depth, const double lo[3], double size, int L_f,
                               int64_t K, int nranks, int rank, int level, int64_t *recv_off, int64_t *send_off,
                               int64_t *recv_box, int64_t *send_box) {
  using namespace hfmm;
  if (!xyz || !lo || !recv_off || !send_off || nranks < 1 || rank < 0 || rank >= nranks || L_f < 2 || L_f > depth ||
      level < 2 || level > L_f || K <= 0)
    return HFMM_E_ARG;
  Tree t;
  std::string err;
  int rc = build_tree(xyz, n, depth, lo, size, t, err);
  if (rc) return rc;
  std::vector<int64_t> cut;
  partition_level2(t, L_f, K, nranks, cut);
  std::vector<int64_t> rlo(cut.begin(), cut.end() - 1), rhi(cut.begin() + 1, cut.end());
  for (int l = 2; l < level; ++l)   // descend to `level` (children ranges are contiguous)
    for (int q = 0; q < nranks; ++q)
      rlo[q] = t.levels[l].child_begin[rlo[q]], rhi[q] = t.levels[l].child_begin[rhi[q]];
  std::vector<std::vector<int64_t>> snd, rcv;
  m2l_halo_lists(t, level, rlo, rhi, rank, snd, rcv);
  recv_off[0] = send_off[0] = 0;
  for (int q = 0; q < nranks; ++q) {
    recv_off[q + 1] = recv_off[q] + (int64_t)rcv[q].size();
    send_off[q + 1] = send_off[q] + (int64_t)snd[q].size();
    if (recv_box) std::copy(rcv[q].begin(), rcv[q].end(), recv_box + recv_off[q]);
    if (send_box) std::copy(snd[q].begin(), snd[q].end(), send_box + send_off[q]);
  }
  return 0;
}
