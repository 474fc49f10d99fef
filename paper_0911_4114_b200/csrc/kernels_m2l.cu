// M2L, the diagonal transfer pass, product code, sm_100a:
//     I_l[alpha][k] = sum_{beta in I(alpha)} T_l[o(beta - alpha)][k] M_l[beta][k]
//
// Sibling-group design.  Targets are processed in groups (the <= 8 children of one parent, or 8
// consecutive boxes): the group's interaction lists are merged into one list of source boxes,
// each source carrying the table id (offset 0..315, or -1) it has for every target of the group.
// A warp owns one group and a chunk of 32 directions k (lane = k), keeps the 8 target
// accumulators in registers and walks the merged source list: every M[beta][k] is loaded once per
// group (coalesced, 512 B per warp) and used for all its targets; the tables of the chunk,
// T[o][k0..k0+31] for all 316 offsets (162 KB), sit in shared memory, read conflict-free with
// lanes over k.  Work units are (k-chunk, group range) in chunk-major order over persistent CTAs,
// so the CTAs running at any time share one chunk: its slice of M (nbox x 32 x 16 B) and of the
// tables stay L2-resident and every M value crosses HBM about once.  One shared-memory table load
// per complex MAC bounds the kernel at ~50% of the FP64 pipe (128 B/clk/SM shared vs 2 DFMA
// warp-instructions/clk/SM).
//
// Tables: explicit [316][K] (operator entry point, random tables) or the 34 canonical tables
// + reflection permutations of the matvec (NEXT 3): T_o[k] = T34[c(o)][perm[op(o)][k]].
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <set>
#include <vector>

#include "hfmm_impl.h"

namespace hfmm {

constexpr int M2LG_KC = 32;       // directions per chunk (lanes)
#ifndef HFMM_M2L_WARPS
#define HFMM_M2L_WARPS 16
#endif
#ifndef HFMM_M2L_PF
#define HFMM_M2L_PF 4
#endif
constexpr int M2LG_WARPS = HFMM_M2L_WARPS;  // groups in flight per CTA (one CTA per SM: 162 KB table chunk)
constexpr int M2LG_NOFF = 316;

__constant__ int32_t c_sym_of[M2LG_NOFF];  // offset id -> canonical id << 4 | op (34-table mode)

__device__ __forceinline__ double2 g_cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

__global__ void __launch_bounds__(32 * M2LG_WARPS, 1) m2l_group_kernel(
    int64_t K, int64_t ngroups, int64_t groups_per_unit, int64_t nunits,
    const int32_t *__restrict__ gtarget /*[G][8]*/, const int32_t *__restrict__ gsrc_row /*[G+1]*/,
    const int32_t *__restrict__ src_box, const int16_t *__restrict__ tid8 /*[E][8]*/,
    const double2 *__restrict__ T, const int32_t *__restrict__ perm /*nullptr: explicit 316 tables*/,
    const double2 *__restrict__ M, double2 *__restrict__ I) {
  extern __shared__ double2 Ts[];  // [316][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (K + M2LG_KC - 1) / M2LG_KC;
  const int64_t ranges = (nunits + nchunks - 1) / nchunks;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t chunk = u / ranges, range = u % ranges;
    const int64_t k0 = chunk * M2LG_KC;
    const int64_t k = k0 + lane;
    const bool kval = k < K;
    __syncthreads();  // previous unit done with Ts
    for (int i = threadIdx.x; i < M2LG_NOFF * M2LG_KC; i += blockDim.x) {
      const int o = i / M2LG_KC, kk = i % M2LG_KC;
      const int64_t kg = k0 + kk;
      double2 v = make_double2(0.0, 0.0);
      if (kg < K) {
        if (perm) {
          const int32_t code = c_sym_of[o];
          v = T[(int64_t)(code >> 4) * K + perm[(int64_t)(code & 15) * K + kg]];
        } else {
          v = T[(int64_t)o * K + kg];
        }
      }
      Ts[i] = v;
    }
    __syncthreads();
    const int64_t g0 = range * groups_per_unit, g1 = min(ngroups, g0 + groups_per_unit);
    for (int64_t g = g0 + warp; g < g1; g += M2LG_WARPS) {
      double2 acc[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[a] = make_double2(0.0, 0.0);
      const int32_t e0 = gsrc_row[g], e1 = gsrc_row[g + 1];
      // sources in batches of PF: all loads of a batch in flight before its MACs
      constexpr int PF = HFMM_M2L_PF;
      for (int32_t e = e0; e < e1; e += PF) {
        double2 m[PF];
        int4 pk[PF];
#pragma unroll
        for (int j = 0; j < PF; ++j) {
          const bool v = e + j < e1;
          m[j] = (v && kval) ? __ldg(&M[(int64_t)src_box[e + j] * K + k]) : make_double2(0.0, 0.0);
          pk[j] = v ? __ldg(reinterpret_cast<const int4 *>(tid8) + e + j) : make_int4(-1, -1, -1, -1);
        }
#pragma unroll
        for (int j = 0; j < PF; ++j) {
          const int16_t *t8 = reinterpret_cast<const int16_t *>(&pk[j]);
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const int t = t8[a];
            if (t >= 0) acc[a] = g_cfma(Ts[t * M2LG_KC + lane], m[j], acc[a]);
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int32_t b = gtarget[g * 8 + a];
        if (b >= 0 && kval) I[(int64_t)b * K + k] = acc[a];
      }
    }
  }
}

// ---- host plan -----------------------------------------------------------------------------------
struct M2LGroupPlan {
  int64_t nbox = 0, K = 0, ngroups = 0, nentries = 0;
  int32_t *gtarget = nullptr, *gsrc_row = nullptr, *src_box = nullptr;
  int16_t *tid8 = nullptr;
};

static void upload_sym_table() {  // __constant__ memory is per device: upload once per device
  static std::set<int> done;
  int d = 0;
  cudaGetDevice(&d);
  if (done.count(d)) return;
  std::vector<int> cids, sym_of;
  canonical_offsets(cids, sym_of);
  std::vector<int32_t> v(sym_of.begin(), sym_of.end());
  cudaMemcpyToSymbol(c_sym_of, v.data(), sizeof(int32_t) * M2LG_NOFF);
  done.insert(d);
}

// targets [box0, box1) of a level with interaction CSR (row / src / oid: host, row indexed by box
// id, oid = offset id 0..315); groups = [gbeg[i], gbeg[i+1]) (<= 8 boxes each) or blocks of 8.
M2LGroupPlan *m2l_group_plan_create(int64_t nbox, int64_t K, const int32_t *row, const int32_t *src,
                                    const int32_t *oid, const std::vector<int64_t> *gbeg) {
  auto *pl = new M2LGroupPlan();
  pl->nbox = nbox, pl->K = K;
  std::vector<int64_t> gb;
  if (gbeg) {
    gb = *gbeg;
  } else {
    for (int64_t b = 0; b < nbox; b += 8) gb.push_back(b);
    gb.push_back(nbox);
  }
  const int64_t G = (int64_t)gb.size() - 1;
  std::vector<int32_t> gt((size_t)G * 8, -1), grow(1, 0), sbox;
  std::vector<int16_t> t8;
  std::vector<int32_t> slot;  // source box -> entry of the current group
  std::vector<int32_t> touched;
  for (int64_t g = 0; g < G; ++g) {
    touched.clear();
    const int64_t base = (int64_t)sbox.size();
    for (int64_t b = gb[g]; b < gb[g + 1]; ++b) {
      const int a = (int)(b - gb[g]);
      gt[(size_t)g * 8 + a] = (int32_t)b;
      for (int32_t e = row[b]; e < row[b + 1]; ++e) {
        const int32_t s = src[e];
        if ((int64_t)slot.size() <= s) slot.resize((size_t)s + 1, -1);
        if (slot[s] < 0) {
          slot[s] = (int32_t)(sbox.size() - base);
          touched.push_back(s);
          sbox.push_back(s);
          t8.insert(t8.end(), 8, (int16_t)-1);
        }
        t8[(size_t)(base + slot[s]) * 8 + a] = (int16_t)oid[e];
      }
    }
    for (int32_t s : touched) slot[s] = -1;
    grow.push_back((int32_t)sbox.size());
  }
  pl->ngroups = G;
  pl->nentries = (int64_t)sbox.size();
  auto up = [](const void *h, size_t bytes) -> void * {
    void *d = nullptr;
    if (bytes && cudaMalloc(&d, bytes) == cudaSuccess) cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    return d;
  };
  pl->gtarget = (int32_t *)up(gt.data(), gt.size() * 4);
  pl->gsrc_row = (int32_t *)up(grow.data(), grow.size() * 4);
  pl->src_box = (int32_t *)up(sbox.data(), sbox.size() * 4);
  pl->tid8 = (int16_t *)up(t8.data(), t8.size() * 2);
  return pl;
}

void m2l_group_plan_destroy(M2LGroupPlan *pl) {
  if (!pl) return;
  for (void *p : {(void *)pl->gtarget, (void *)pl->gsrc_row, (void *)pl->src_box, (void *)pl->tid8})
    if (p) cudaFree(p);
  delete pl;
}

void m2l_group_apply(const M2LGroupPlan *pl, const double2 *T, const int32_t *perm, const double2 *M, double2 *I,
                     cudaStream_t s) {
  if (!pl || pl->ngroups <= 0 || pl->K <= 0) return;
  if (perm) upload_sym_table();
  const size_t smem = (size_t)M2LG_NOFF * M2LG_KC * sizeof(double2);
  cudaFuncSetAttribute(m2l_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nchunks = (pl->K + M2LG_KC - 1) / M2LG_KC;
  // group ranges per chunk: one chunk spread over all SMs at a time (chunk-major units), so the
  // chunk's slice of M stays L2-resident while every CTA works on it; >= 8 groups per unit
  int64_t ranges = std::max<int64_t>(1, std::min<int64_t>((pl->ngroups + M2LG_WARPS - 1) / M2LG_WARPS, nsm));
  const int64_t gpu = (pl->ngroups + ranges - 1) / ranges;
  ranges = (pl->ngroups + gpu - 1) / gpu;
  const int64_t nunits = nchunks * ranges;
  const unsigned grid = (unsigned)std::min<int64_t>(nunits, nsm);
  m2l_group_kernel<<<grid, 32 * M2LG_WARPS, smem, s>>>(pl->K, pl->ngroups, gpu, nunits, pl->gtarget, pl->gsrc_row,
                                                       pl->src_box, pl->tid8, T, perm, M, I);
}

}  // namespace hfmm
