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
// Parent-block variant (m2l_dense_kernel, used when a group's targets are the children of one
// parent P and its lists are the standard ones): the sources are the children e of the 26
// neighbour parents P + D, and target d / source (D, e) have offset o = 2D + e - d.  All 64
// (d, e) pairs of one neighbour parent with the same delta = e - d share one table T[2D + delta]
// (admissible iff |2D + delta|_inf >= 2), so one shared-memory table load serves 1..8 MACs
// (an interior group: 702 table loads for 1,664 MACs instead of 1,512 for 1,512) with no
// per-pair index or branch work.  Both variants compute exactly the CSR's terms; the plan proves
// the equivalence per group (else it keeps the list variant).
//
// Tables: explicit [316][K] (operator entry point, random tables) or the 34 canonical tables
// + reflection permutations of the matvec (NEXT 3): T_o[k] = T34[c(o)][perm[op(o)][k]].
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
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
#ifndef HFMM_M2L_SPLIT
#define HFMM_M2L_SPLIT 0  // parent-block kernel: real/imaginary halves of each MAC in separate accumulators
#endif
#ifndef HFMM_M2L_L1PF
#define HFMM_M2L_L1PF 0  // parent-block kernel: prefetch the next neighbour parent's sources into L1
#endif
#ifndef HFMM_M2L_DPF
#define HFMM_M2L_DPF 0  // parent-block kernel: prefetch the next neighbour parent's sources
#endif
constexpr int M2LG_WARPS = HFMM_M2L_WARPS;  // groups in flight per CTA (one CTA per SM: 162 KB table chunk)
constexpr int M2LG_NOFF = 316;

__constant__ int32_t c_sym_of[M2LG_NOFF];  // offset id -> canonical id << 4 | op (34-table mode)

__device__ __forceinline__ double2 g_cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

// c_slot_id[s] = offset id of the cube position s = (ox+3)*49 + (oy+3)*7 + (oz+3), o in [-3,3]^3,
// or -1 for the 27 adjacent offsets |o|_inf <= 1 (parent-block kernel: their tables are zero)
constexpr int M2LB_SLOTS = 343;
__constant__ int16_t c_slot_id[M2LB_SLOTS];
#ifndef HFMM_M2L_SKIP
#define HFMM_M2L_SKIP 0  // parent-block kernel: skip the zero tables of adjacent slots (warp-uniform branch;
                         // A/B: B64 50.0 vs 41.8 ms, the branches split the scheduled MAC stream -> off)
#endif
// c_zero_dl[D] bit dl: neighbour parent D = (Dx,Dy,Dz) + 1 in base 3 and child offset delta = e - d
// (dl in base 3) give an adjacent offset 2D + delta (|.|_inf <= 1), whose table is zero
__constant__ uint32_t c_zero_dl[27];

__device__ __forceinline__ void fill_tables(double2 *Ts, const double2 *__restrict__ T, const int32_t *__restrict__ perm,
                                            int64_t K, int64_t k0) {
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
    fill_tables(Ts, T, perm, K, k0);
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

// Child slot c = x << 2 | y << 1 | z of a box inside its parent.  gtarget [G][8] by child slot d,
// gsrc [G][27][8] by neighbour-parent slot D and child slot e (-1: no box), gmask [G] bit D set
// when parent slot D holds a source.  The chunk's tables sit in shared memory by cube position
// (343 slots, 176 KB) with zero tables at the adjacent offsets, so every (D, delta) reads
// T[2D + delta] at a compile-time offset from a per-D base and all 64 (d, e) pairs of a
// neighbour parent run without branches (the adjacent pairs add exact zeros: 9% extra MACs for an
// interior group, 1,664 issued for 1,512 terms).
__device__ __forceinline__ void fill_tables_cube(double2 *Ts, const double2 *__restrict__ T,
                                                 const int32_t *__restrict__ perm, int64_t K, int64_t k0) {
  for (int i = threadIdx.x; i < M2LB_SLOTS * M2LG_KC; i += blockDim.x) {
    const int sl = i / M2LG_KC, kk = i % M2LG_KC;
    const int o = c_slot_id[sl];
    const int64_t kg = k0 + kk;
    double2 v = make_double2(0.0, 0.0);
    if (o >= 0 && kg < K) {
      if (perm) {
        const int32_t code = c_sym_of[o];
        v = T[(int64_t)(code >> 4) * K + perm[(int64_t)(code & 15) * K + kg]];
      } else {
        v = T[(int64_t)o * K + kg];
      }
    }
    Ts[i] = v;
  }
}

__global__ void __launch_bounds__(32 * M2LG_WARPS, 1) m2l_dense_kernel(
    int64_t K, int64_t ngroups, int64_t groups_per_unit, int64_t nunits, const int32_t *__restrict__ gtarget,
    const int32_t *__restrict__ gsrc, const uint32_t *__restrict__ gmask, const double2 *__restrict__ T,
    const int32_t *__restrict__ perm, const double2 *__restrict__ M, double2 *__restrict__ I) {
  extern __shared__ double2 Ts[];  // [343][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (K + M2LG_KC - 1) / M2LG_KC;
  const int64_t ranges = (nunits + nchunks - 1) / nchunks;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t chunk = u / ranges, range = u % ranges;
    const int64_t k0 = chunk * M2LG_KC;
    const int64_t k = k0 + lane;
    const bool kval = k < K;
    __syncthreads();  // previous unit done with Ts
    fill_tables_cube(Ts, T, perm, K, k0);
    __syncthreads();
    const int64_t g0 = range * groups_per_unit, g1 = min(ngroups, g0 + groups_per_unit);
    for (int64_t g = g0 + warp; g < g1; g += M2LG_WARPS) {
      double2 acc[8];
#if HFMM_M2L_SPLIT
      double2 acc2[8];  // second accumulator per target: independent FMA chains (ILP)
#pragma unroll
      for (int a = 0; a < 8; ++a) acc2[a] = make_double2(0.0, 0.0);
#endif
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[a] = make_double2(0.0, 0.0);
      const uint32_t mask = __ldg(&gmask[g]);
      // neighbour parents in mask order; the next parent's 8 source loads are issued before the
      // current parent's MACs (software pipelining across the L2 latency)
      auto load8 = [&](int D, double2 *m) {
        const int4 *sp = reinterpret_cast<const int4 *>(gsrc + (g * 27 + D) * 8);
        const int4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
        const int32_t sid[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          m[e] = (sid[e] >= 0 && kval) ? __ldg(&M[(int64_t)sid[e] * K + k]) : make_double2(0.0, 0.0);
      };
      int D = mask ? __ffs(mask) - 1 : 27;
      double2 m[8];
      if (D < 27) load8(D, m);
      while (D < 27) {
        const uint32_t rest = mask & ~((2u << D) - 1u);
        const int Dn = rest ? __ffs(rest) - 1 : 27;
#if HFMM_M2L_L1PF
        if (Dn < 27 && kval) {  // the next parent's sources into L1 while this parent's MACs run
          const int4 *sp = reinterpret_cast<const int4 *>(gsrc + (g * 27 + Dn) * 8);
          const int4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
          const int32_t sid[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (sid[e] >= 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(&M[(int64_t)sid[e] * K + k]));
        }
#endif
#if HFMM_M2L_DPF
        double2 mn[8];
        if (Dn < 27) load8(Dn, mn);
#endif
        // T[2D + delta] = Tb[delta slot offset]: base at cube position 2D + (-1,-1,-1)
        const int Dx = D / 9 - 1, Dy = (D / 3) % 3 - 1, Dz = D % 3 - 1;
        const double2 *Tb = Ts + ((2 * Dx + 2) * 49 + (2 * Dy + 2) * 7 + (2 * Dz + 2)) * M2LG_KC + lane;
#if HFMM_M2L_SKIP
        const uint32_t zm = c_zero_dl[D];  // warp-uniform: bit dl set when slot 2D + delta is adjacent
#endif
#pragma unroll
        for (int dl = 0; dl < 27; ++dl) {
          const int dx = dl / 9 - 1, dy = (dl / 3) % 3 - 1, dz = dl % 3 - 1;
#if HFMM_M2L_SKIP
          if ((zm >> dl) & 1u) continue;  // zero table: skip its load and its MACs
#endif
          const double2 t = Tb[((dx + 1) * 49 + (dy + 1) * 7 + (dz + 1)) * M2LG_KC];
#pragma unroll
          for (int d = 0; d < 8; ++d) {
            const int ex = (d >> 2) + dx, ey = ((d >> 1) & 1) + dy, ez = (d & 1) + dz;
            if (ex < 0 || ex > 1 || ey < 0 || ey > 1 || ez < 0 || ez > 1) continue;
#if HFMM_M2L_SPLIT
            const double2 mm = m[(ex << 2) | (ey << 1) | ez];
            acc[d] = make_double2(fma(t.x, mm.x, acc[d].x), fma(t.x, mm.y, acc[d].y));
            acc2[d] = make_double2(fma(-t.y, mm.y, acc2[d].x), fma(t.y, mm.x, acc2[d].y));
#else
            acc[d] = g_cfma(t, m[(ex << 2) | (ey << 1) | ez], acc[d]);
#endif
          }
        }
#if HFMM_M2L_DPF
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = mn[e];
#else
        if (Dn < 27) load8(Dn, m);
#endif
        D = Dn;
      }
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const int32_t b = gtarget[g * 8 + d];
#if HFMM_M2L_SPLIT
        acc[d] = make_double2(acc[d].x + acc2[d].x, acc[d].y + acc2[d].y);
#endif
        if (b >= 0 && kval) I[(int64_t)b * K + k] = acc[d];
      }
    }
  }
}

// Two sibling groups per warp (GPW = 2): the tables depend only on the offset 2D + delta, so one
// shared-memory table load serves the MACs of both groups (half the table traffic per MAC, twice
// the accumulators in registers); neighbour parents of either group's mask, a missing parent's
// sources are zeros.  M2LB2_WARPS warps x 2 groups per CTA.
#ifndef HFMM_M2L_GPW
#define HFMM_M2L_GPW 1   // 2: m2l_dense2_kernel (A/B: B64 52 vs 42 ms, kept off)
#endif
constexpr int M2LB2_WARPS = 8;

__global__ void __launch_bounds__(32 * M2LB2_WARPS, 1) m2l_dense2_kernel(
    int64_t K, int64_t ngroups, int64_t groups_per_unit, int64_t nunits, const int32_t *__restrict__ gtarget,
    const int32_t *__restrict__ gsrc, const uint32_t *__restrict__ gmask, const double2 *__restrict__ T,
    const int32_t *__restrict__ perm, const double2 *__restrict__ M, double2 *__restrict__ I) {
  extern __shared__ double2 Ts[];  // [343][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nchunks = (K + M2LG_KC - 1) / M2LG_KC;
  const int64_t ranges = (nunits + nchunks - 1) / nchunks;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t chunk = u / ranges, range = u % ranges;
    const int64_t k0 = chunk * M2LG_KC;
    const int64_t k = k0 + lane;
    const bool kval = k < K;
    __syncthreads();  // previous unit done with Ts
    fill_tables_cube(Ts, T, perm, K, k0);
    __syncthreads();
    const int64_t g0 = range * groups_per_unit, g1 = min(ngroups, g0 + groups_per_unit);
    for (int64_t ga = g0 + 2 * warp; ga < g1; ga += 2 * M2LB2_WARPS) {
      const int64_t gb = ga + 1;
      const bool hb = gb < g1;
      double2 acc[2][8];
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[0][a] = acc[1][a] = make_double2(0.0, 0.0);
      const uint32_t mka = __ldg(&gmask[ga]), mkb = hb ? __ldg(&gmask[gb]) : 0u;
      const uint32_t mask = mka | mkb;
      auto load8 = [&](int64_t g, bool has, int D, double2 *m) {
        if (!has) {
#pragma unroll
          for (int e = 0; e < 8; ++e) m[e] = make_double2(0.0, 0.0);
          return;
        }
        const int4 *sp = reinterpret_cast<const int4 *>(gsrc + (g * 27 + D) * 8);
        const int4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
        const int32_t sid[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e)
          m[e] = (sid[e] >= 0 && kval) ? __ldg(&M[(int64_t)sid[e] * K + k]) : make_double2(0.0, 0.0);
      };
      int D = mask ? __ffs(mask) - 1 : 27;
      double2 m[2][8];
      if (D < 27) load8(ga, (mka >> D) & 1u, D, m[0]), load8(gb, (mkb >> D) & 1u, D, m[1]);
      while (D < 27) {
        const uint32_t rest = mask & ~((2u << D) - 1u);
        const int Dn = rest ? __ffs(rest) - 1 : 27;
        const int Dx = D / 9 - 1, Dy = (D / 3) % 3 - 1, Dz = D % 3 - 1;
        const double2 *Tb = Ts + ((2 * Dx + 2) * 49 + (2 * Dy + 2) * 7 + (2 * Dz + 2)) * M2LG_KC + lane;
#pragma unroll
        for (int dl = 0; dl < 27; ++dl) {
          const int dx = dl / 9 - 1, dy = (dl / 3) % 3 - 1, dz = dl % 3 - 1;
          const double2 t = Tb[((dx + 1) * 49 + (dy + 1) * 7 + (dz + 1)) * M2LG_KC];
#pragma unroll
          for (int d = 0; d < 8; ++d) {
            const int ex = (d >> 2) + dx, ey = ((d >> 1) & 1) + dy, ez = (d & 1) + dz;
            if (ex < 0 || ex > 1 || ey < 0 || ey > 1 || ez < 0 || ez > 1) continue;
            const int e = (ex << 2) | (ey << 1) | ez;
            acc[0][d] = g_cfma(t, m[0][e], acc[0][d]);
            acc[1][d] = g_cfma(t, m[1][e], acc[1][d]);
          }
        }
        if (Dn < 27) load8(ga, (mka >> Dn) & 1u, Dn, m[0]), load8(gb, (mkb >> Dn) & 1u, Dn, m[1]);
        D = Dn;
      }
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const int32_t ba = gtarget[ga * 8 + d];
        if (ba >= 0 && kval) I[(int64_t)ba * K + k] = acc[0][d];
        if (hb) {
          const int32_t bb = gtarget[gb * 8 + d];
          if (bb >= 0 && kval) I[(int64_t)bb * K + k] = acc[1][d];
        }
      }
    }
  }
}

// Parent-block kernel with the next neighbour parent's sources prefetched (m2l_dense_pf_kernel,
// HFMM_M2L_PF16): chunks of 16 directions; a warp runs two sibling groups, lanes 0-15 one and
// 16-31 the other, over the same 16 directions, so every table read is a 2-way broadcast (half the
// shared-memory wavefronts per MAC of the 32-direction kernel, half its table footprint: 88 KB); the
// 8 source values of the next neighbour parent are fetched with cp.async into a per-warp double
// buffer in shared memory while the current parent's MACs run (the 32-direction kernel exposes that
// L2 latency: long-scoreboard stalls, profiles/r01), without holding them in registers.
#ifndef HFMM_M2L_PF16
#define HFMM_M2L_PF16 0   // A/B (profiles/r02/m2l_pf16_ab.txt): B64 44.7 vs 41.9 ms for the 32-direction kernel
#endif
constexpr int M2LP_KC = 16, M2LP_WARPS = 16;

__device__ __forceinline__ void m2l_cp_async16(double2 *smem, const double2 *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;   // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void fill_tables_cube16(double2 *Ts, const double2 *__restrict__ T,
                                                   const int32_t *__restrict__ perm, int64_t K, int64_t k0) {
  for (int i = threadIdx.x; i < M2LB_SLOTS * M2LP_KC; i += blockDim.x) {
    const int sl = i / M2LP_KC, kk = i % M2LP_KC;
    const int o = c_slot_id[sl];
    const int64_t kg = k0 + kk;
    double2 v = make_double2(0.0, 0.0);
    if (o >= 0 && kg < K) {
      if (perm) {
        const int32_t code = c_sym_of[o];
        v = T[(int64_t)(code >> 4) * K + perm[(int64_t)(code & 15) * K + kg]];
      } else {
        v = T[(int64_t)o * K + kg];
      }
    }
    Ts[i] = v;
  }
}

__global__ void __launch_bounds__(32 * M2LP_WARPS, 1) m2l_dense_pf_kernel(
    int64_t K, int64_t ngroups, int64_t groups_per_unit, int64_t nunits, const int32_t *__restrict__ gtarget,
    const int32_t *__restrict__ gsrc, const uint32_t *__restrict__ gmask, const double2 *__restrict__ T,
    const int32_t *__restrict__ perm, const double2 *__restrict__ M, double2 *__restrict__ I) {
  extern __shared__ double2 Ts[];                          // [343][16] tables, then [warps][2][8][32] buffers
  double2 *bufs = Ts + M2LB_SLOTS * M2LP_KC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = lane >> 4;
  double2 *wb = bufs + warp * (2 * 8 * 32);
  const int64_t nchunks = (K + M2LP_KC - 1) / M2LP_KC;
  const int64_t ranges = (nunits + nchunks - 1) / nchunks;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t chunk = u / ranges, range = u % ranges;
    const int64_t k0 = chunk * M2LP_KC;
    const int64_t k = k0 + (lane & 15);
    const bool kval = k < K;
    __syncthreads();  // previous unit done with Ts
    fill_tables_cube16(Ts, T, perm, K, k0);
    __syncthreads();
    const int64_t g0 = range * groups_per_unit, g1 = min(ngroups, g0 + groups_per_unit);
    for (int64_t gp = g0 + 2 * warp; gp < g1; gp += 2 * M2LP_WARPS) {
      const int64_t g = gp + half;                         // this half-warp's group
      const bool hg = g < g1;
      double2 acc[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) acc[a] = make_double2(0.0, 0.0);
      const uint32_t mk = hg ? __ldg(&gmask[g]) : 0u;
      const uint32_t mask = mk | __shfl_xor_sync(0xffffffffu, mk, 16);   // union over the two groups
      auto issue = [&](int D, int stage) {                 // 8 source values of parent slot D
        const bool has = (mk >> D) & 1u;
        const int32_t *sp = gsrc + (g * 27 + D) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int32_t sid = has ? __ldg(&sp[e]) : -1;
          const bool ok = sid >= 0 && kval;
          m2l_cp_async16(&wb[(stage * 8 + e) * 32 + lane], ok ? &M[(int64_t)sid * K + k] : M, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::);
      };
      int D = mask ? __ffs(mask) - 1 : 27;
      int stage = 0;
      if (D < 27) issue(D, 0);
      while (D < 27) {
        const uint32_t rest = mask & ~((2u << D) - 1u);
        const int Dn = rest ? __ffs(rest) - 1 : 27;
        if (Dn < 27) {
          issue(Dn, stage ^ 1);
          asm volatile("cp.async.wait_group 1;\n" ::);   // the current stage has landed
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        double2 m[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = wb[(stage * 8 + e) * 32 + lane];
        const int Dx = D / 9 - 1, Dy = (D / 3) % 3 - 1, Dz = D % 3 - 1;
        const double2 *Tb = Ts + ((2 * Dx + 2) * 49 + (2 * Dy + 2) * 7 + (2 * Dz + 2)) * M2LP_KC + (lane & 15);
#pragma unroll
        for (int dl = 0; dl < 27; ++dl) {
          const int dx = dl / 9 - 1, dy = (dl / 3) % 3 - 1, dz = dl % 3 - 1;
          const double2 t = Tb[((dx + 1) * 49 + (dy + 1) * 7 + (dz + 1)) * M2LP_KC];
#pragma unroll
          for (int d = 0; d < 8; ++d) {
            const int ex = (d >> 2) + dx, ey = ((d >> 1) & 1) + dy, ez = (d & 1) + dz;
            if (ex < 0 || ex > 1 || ey < 0 || ey > 1 || ez < 0 || ez > 1) continue;
            acc[d] = g_cfma(t, m[(ex << 2) | (ey << 1) | ez], acc[d]);
          }
        }
        stage ^= 1;
        D = Dn;
      }
      if (hg) {
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const int32_t b = gtarget[g * 8 + d];
          if (b >= 0 && kval) I[(int64_t)b * K + k] = acc[d];
        }
      }
    }
  }
}

// ---- host plan -----------------------------------------------------------------------------------
struct M2LGroupPlan {
  int64_t nbox = 0, K = 0, ngroups = 0, nentries = 0;
  int32_t *gtarget = nullptr, *gsrc_row = nullptr, *src_box = nullptr;
  int16_t *tid8 = nullptr;
  // parent-block variant (dense == true): targets by child slot, sources by (parent slot, child slot)
  bool dense = false;
  int64_t dense_macs = 0;  // MACs the parent-block kernel issues (>= nentries)
  int32_t *dtarget = nullptr, *dsrc = nullptr;
  uint32_t *dmask = nullptr;
};

// ---- parent-block M2L on the FP64 tensor core (DMMA m8n8k4) -----------------------------------
// For one direction k and one neighbour-parent slot D the parent-block sum is a matrix product
// shared by every sibling group:  I[d][g] += sum_e A_{D,k}[d][e] B_{D,k}[e][g],  A[d][e] =
// T[2D + e - d][k] (8 x 8, zero at adjacent offsets), B[e][g] = M[child e of (P_g + D)][k].
// A warp runs it for a direction pair (k, k + 1) and a batch of 8 groups as real 8 x 8 x 4
// DMMAs (mma.sync.m8n8k4.f64: thread t holds A[t/4][t%4], B[t%4][t/4], C[t/4][2(t%4) + j]):
//   C_re += A_re B_re - A_im B_im,   C_im += A_re B_im + A_im B_re   (two k-steps over e)
// 16 DMMAs (4,096 FMAs) per (D, pair, batch) replace 512 DFMA warp-instructions: the MACs issue as
// a few dozen instructions and never read three vector registers per FMA (the DFMA kernel's
// issue / register-port ceiling, DESIGN 6.1).  B200's DMMA and DFMA share one FP64 pipe
// (profiles/r02/dmma_probe.txt: 37.1 TFLOP/s DMMA alone), so the gain would be the issue side.
// Measured (same box, C2 B64): 78 ms with B fragments loaded from global memory (L1TEX 94% busy:
// 32 rows per warp load), 69 ms with the batch's source ids staged, 62.7 ms with the sources
// staged by cp.async (tensor pipe 39% active; stalls: DMMA dependency waits, shared-memory
// scoreboards, 12 warps/SM; split accumulators, 8 chains per warp: 65.2 ms) vs 41.7 ms for the
// DFMA parent-block kernel: kept off (parity-green).
// Tables: the chunk's [M2LD_KC directions][343 cube slots] k-major in shared memory (a warp reads
// 32 different slots of one direction: no bank conflicts), M from global / L2 as 32-byte (k, k+1)
// pairs.  Same plan data (dtarget / dsrc / dmask) and the same terms as m2l_dense_kernel.
#ifndef HFMM_M2L_DMMA
#define HFMM_M2L_DMMA 0   // A/B (profiles/r02/m2l_dmma_ab.txt): B64 62.7 vs 41.7 ms for the DFMA kernel -> off
#endif
constexpr int M2LD_KC = 8;       // directions per table chunk (4 direction pairs = 4 warps)
constexpr int M2LD_WARPS = M2LD_KC / 2;
constexpr int M2LD_MP = M2LD_KC + 1;   // staged-source row pitch (complex values): conflict-free B reads

__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void m2ld_cp16(double2 *smem, const double2 *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

__device__ __forceinline__ void fill_tables_kmajor(double2 *Ts, const double2 *__restrict__ T,
                                                   const int32_t *__restrict__ perm, int64_t K, int64_t k0) {
  // Ts[kk][sl] = T_{o(sl)}[k0 + kk]; consecutive threads take consecutive directions of one slot
  for (int i = threadIdx.x; i < M2LB_SLOTS * M2LD_KC; i += blockDim.x) {
    const int sl = i / M2LD_KC, kk = i % M2LD_KC;
    const int o = c_slot_id[sl];
    const int64_t kg = k0 + kk;
    double2 v = make_double2(0.0, 0.0);
    if (o >= 0 && kg < K) {
      if (perm) {
        const int32_t code = c_sym_of[o];
        v = T[(int64_t)(code >> 4) * K + perm[(int64_t)(code & 15) * K + kg]];
      } else {
        v = T[(int64_t)o * K + kg];
      }
    }
    Ts[kk * M2LB_SLOTS + sl] = v;
  }
}

// Sources of one neighbour-parent slot D for the batch's 8 groups: the CTA stages
// Ms[g * 8 + e][kk] = M[child e of (P_g + D)][k0 + kk] (kk < M2LD_KC; 128-byte rows, cp.async,
// zeros for missing children) so the DMMA B fragments come from shared memory -- loading them
// straight from global memory put 32 different rows under every warp load (8x the L1
// wavefronts of the DFMA kernel; ncu: L1TEX at 94% and the tensor pipe at 35%).
__device__ __forceinline__ void m2ld_stage(double2 *Ms, const int32_t *sid_s, int D, const double2 *__restrict__ M,
                                           int64_t K, int64_t k0) {
  for (int i = threadIdx.x; i < 64 * M2LD_KC; i += blockDim.x) {
    const int row = i / M2LD_KC, kk = i % M2LD_KC;
    const int g = row >> 3, e = row & 7;
    const int32_t sid = sid_s[(g * 27 + D) * 8 + e];
    double2 *dst = Ms + row * M2LD_MP + kk;
    if (sid >= 0 && k0 + kk < K) m2ld_cp16(dst, M + (int64_t)sid * K + k0 + kk);
    else *dst = make_double2(0.0, 0.0);
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

__global__ void __launch_bounds__(32 * M2LD_WARPS, 3) m2l_dmma_kernel(
    int64_t K, int64_t ngroups, int64_t batches_per_unit, int64_t nunits, const int32_t *__restrict__ gtarget,
    const int32_t *__restrict__ gsrc, const uint32_t *__restrict__ gmask, const double2 *__restrict__ T,
    const int32_t *__restrict__ perm, const double2 *__restrict__ M, double2 *__restrict__ I) {
  extern __shared__ double2 Ts[];  // [M2LD_KC][343] tables, [2][64][M2LD_MP] staged sources, source ids
  double2 *Ms = Ts + M2LB_SLOTS * M2LD_KC;
  int32_t *sid_s = reinterpret_cast<int32_t *>(Ms + 2 * 64 * M2LD_MP);  // [8 groups][27][8]
  __shared__ uint32_t mask_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, c = lane & 3;   // fragment row / column of this thread
  const int64_t nchunks = (K + M2LD_KC - 1) / M2LD_KC;
  const int64_t nbatch = (ngroups + 7) / 8;
  const int64_t ranges = (nunits + nchunks - 1) / nchunks;
  // A[d = r][e = c + 4 s]: offset delta = e - d in child units
  const int dx0 = -(r >> 2), dy0 = -((r >> 1) & 1), dz0 = -(r & 1);
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t chunk = u / ranges, range = u % ranges;
    const int64_t kbase = chunk * M2LD_KC;
    __syncthreads();  // previous unit done with Ts
    fill_tables_kmajor(Ts, T, perm, K, kbase);
    const int kk = 2 * warp;                      // this warp's direction pair (kbase + kk, + 1)
    const int64_t k = kbase + kk;
    const bool kv0 = k < K, kv1 = k + 1 < K;
    const int64_t b0 = range * batches_per_unit, b1 = min(nbatch, b0 + batches_per_unit);
    for (int64_t bt = b0; bt < b1; ++bt) {
      __syncthreads();  // tables filled / previous batch done with sid_s and Ms
      for (int i = threadIdx.x; i < 8 * 27 * 8; i += blockDim.x) {
        const int64_t g = bt * 8 + i / (27 * 8);
        sid_s[i] = g < ngroups ? __ldg(&gsrc[bt * 8 * 27 * 8 + i]) : -1;
      }
      if (warp == 0) {
        const uint32_t m = (lane < 8 && bt * 8 + lane < ngroups) ? __ldg(&gmask[bt * 8 + lane]) : 0u;
        const uint32_t all = __reduce_or_sync(0xffffffffu, m);
        if (lane == 0) mask_s = all;
      }
      __syncthreads();
      uint32_t mask = mask_s;
      double cre[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, cim[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [k][j]
      int D = mask ? __ffs(mask) - 1 : 27;
      int buf = 0;
      if (D < 27) m2ld_stage(Ms, sid_s, D, M, K, kbase);
      while (D < 27) {
        const uint32_t rest = mask & ~((2u << D) - 1u);
        const int Dn = rest ? __ffs(rest) - 1 : 27;
        if (Dn < 27) {   // next parent's sources into the other buffer while this one is used
          m2ld_stage(Ms + (buf ^ 1) * 64 * M2LD_MP, sid_s, Dn, M, K, kbase);
          asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
          asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const double2 *Mb = Ms + buf * 64 * M2LD_MP;
        const int Dx = D / 9 - 1, Dy = (D / 3) % 3 - 1, Dz = D % 3 - 1;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int e = c + 4 * s;
          // A: T[2D + e - d][k, k + 1] from the k-major chunk tables
          const int ox = 2 * Dx + (e >> 2) + dx0, oy = 2 * Dy + ((e >> 1) & 1) + dy0, oz = 2 * Dz + (e & 1) + dz0;
          const int sl = (ox + 3) * 49 + (oy + 3) * 7 + (oz + 3);
          const double2 a0 = Ts[kk * M2LB_SLOTS + sl], a1 = Ts[(kk + 1) * M2LB_SLOTS + sl];
          // B: M[child e of (P_g + D)][k, k + 1], g = r
          const double2 m0 = Mb[(r * 8 + e) * M2LD_MP + kk], m1 = Mb[(r * 8 + e) * M2LD_MP + kk + 1];
          // C_re += A_re B_re - A_im B_im;  C_im += A_re B_im + A_im B_re  (k, then k + 1)
          dmma_8x8x4(cre[0][0], cre[0][1], a0.x, m0.x);
          dmma_8x8x4(cim[0][0], cim[0][1], a0.x, m0.y);
          dmma_8x8x4(cre[1][0], cre[1][1], a1.x, m1.x);
          dmma_8x8x4(cim[1][0], cim[1][1], a1.x, m1.y);
          dmma_8x8x4(cre[0][0], cre[0][1], -a0.y, m0.y);
          dmma_8x8x4(cim[0][0], cim[0][1], a0.y, m0.x);
          dmma_8x8x4(cre[1][0], cre[1][1], -a1.y, m1.y);
          dmma_8x8x4(cim[1][0], cim[1][1], a1.y, m1.x);
        }
        __syncthreads();  // every warp done with this buffer before it is refilled
        buf ^= 1;
        D = Dn;
      }
      // C[d = r][g = 2c + j] -> I[target d of group bt*8 + 2c + j][k, k + 1]
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t g = bt * 8 + 2 * c + j;
        if (g >= ngroups) continue;
        const int32_t b = __ldg(&gtarget[g * 8 + r]);
        if (b < 0) continue;
        if (kv0) I[(int64_t)b * K + k] = make_double2(cre[0][j], cim[0][j]);
        if (kv1) I[(int64_t)b * K + k + 1] = make_double2(cre[1][j], cim[1][j]);
      }
    }
  }
}

#ifndef HFMM_M2L_DENSE_MIN
#define HFMM_M2L_DENSE_MIN 0.5  // use the parent-block kernel when useful / issued MACs >= this
#endif

static void upload_slot_table() {
  std::lock_guard<std::recursive_mutex> lk(cache_mutex());
  static std::set<int> done;
  int d = 0;
  cudaGetDevice(&d);
  if (done.count(d)) return;
  int16_t t[M2LB_SLOTS];
  for (int sl = 0; sl < M2LB_SLOTS; ++sl) {
    const int o[3] = {sl / 49 - 3, (sl / 7) % 7 - 3, sl % 7 - 3};
    const bool adm = std::max(std::abs(o[0]), std::max(std::abs(o[1]), std::abs(o[2]))) >= 2;
    t[sl] = (int16_t)(adm ? offset_id(o[0], o[1], o[2]) : -1);
  }
  cudaMemcpyToSymbol(c_slot_id, t, sizeof(t));
  uint32_t z[27];
  for (int D = 0; D < 27; ++D) {
    const int Dc[3] = {D / 9 - 1, (D / 3) % 3 - 1, D % 3 - 1};
    z[D] = 0;
    for (int dl = 0; dl < 27; ++dl) {
      const int dc[3] = {dl / 9 - 1, (dl / 3) % 3 - 1, dl % 3 - 1};
      bool adj = true;
      for (int c = 0; c < 3; ++c) adj = adj && std::abs(2 * Dc[c] + dc[c]) <= 1;
      if (adj) z[D] |= 1u << dl;
    }
  }
  cudaMemcpyToSymbol(c_zero_dl, z, sizeof(z));
  done.insert(d);
}

// Parent-block form of one group, derived from the CSR alone and proven equivalent to it: the
// targets' relative positions follow from shared sources (o_a(beta) - o_b(beta) = x_b - x_a);
// a choice of child slots d_a in {0,1}^3 places every source at r = d_a + o_a(beta) relative to
// the parent's corner (child units), i.e. neighbour parent D = floor(r / 2) in {-1,0,1}^3 \ {0}
// and child slot e = r - 2D.  Accepted when the placement is consistent and the number of
// admissible (d, D, e) triples over existing boxes equals the group's CSR entries (each entry is
// one such triple with the same offset, so the two sums then have the same terms).
static bool dense_group(int na, const int32_t *tgt, const int32_t *row, const int32_t *src, const int32_t *oid,
                        int32_t dt[8], int32_t ds[27 * 8], uint32_t &mask, int64_t &macs) {
  struct Ent { int a; int32_t s; int o[3]; };
  std::vector<Ent> ents;
  for (int a = 0; a < na; ++a)
    for (int32_t e = row[tgt[a]]; e < row[tgt[a] + 1]; ++e) {
      Ent x{a, src[e], {0, 0, 0}};
      offset_vec(oid[e], x.o);
      ents.push_back(x);
    }
  // relative target positions p_a (p_0 = 0) through shared sources (entries sorted by source)
  std::sort(ents.begin(), ents.end(), [](const Ent &x, const Ent &y) { return x.s < y.s; });
  int p[8][3];
  bool known[8] = {false};
  known[0] = true, p[0][0] = p[0][1] = p[0][2] = 0;
  for (int round = 0; round < 8; ++round) {
    bool changed = false;
    for (size_t i = 0; i < ents.size();) {
      size_t j = i;
      int ref = -1;
      while (j < ents.size() && ents[j].s == ents[i].s) {
        if (ref < 0 && known[ents[j].a]) ref = (int)j;
        ++j;
      }
      if (ref >= 0)
        for (size_t t = i; t < j; ++t)
          if (!known[ents[t].a]) {
            for (int c = 0; c < 3; ++c) p[ents[t].a][c] = p[ents[ref].a][c] + ents[ref].o[c] - ents[t].o[c];
            known[ents[t].a] = changed = true;
          }
      i = j;
    }
    if (!changed) break;
  }
  for (int a = 0; a < na; ++a)
    if (!known[a]) return false;
  for (int c0 = 0; c0 < 8; ++c0) {
    const int d0[3] = {c0 >> 2, (c0 >> 1) & 1, c0 & 1};
    bool ok = true;
    int slot[8];
    int used = 0;
    for (int a = 0; a < na && ok; ++a) {
      int c = 0;
      for (int i = 0; i < 3; ++i) {
        const int v = d0[i] + p[a][i];
        if (v < 0 || v > 1) ok = false;
        c = 2 * c + v;
      }
      if (!ok || (used >> c) & 1) ok = false;
      used |= 1 << c, slot[a] = c;
    }
    if (!ok) continue;
    for (int i = 0; i < 8; ++i) dt[i] = -1;
    for (int i = 0; i < 27 * 8; ++i) ds[i] = -1;
    for (int a = 0; a < na; ++a) dt[slot[a]] = tgt[a];
    mask = 0;
    int32_t prev_s = -1, prev_cell = -1;
    for (const Ent &x : ents) {  // sorted by source: one source, one cell
      int D = 0, e = 0;
      for (int i = 0; i < 3; ++i) {
        const int r = ((slot[x.a] >> (2 - i)) & 1) + x.o[i];
        const int Q = (r >= 0) ? r / 2 : -((1 - r) / 2);  // floor(r / 2)
        if (Q < -1 || Q > 1) ok = false;
        D = 3 * D + (Q + 1), e = 2 * e + (r - 2 * Q);
      }
      if (!ok || D == 13) { ok = false; break; }
      int32_t &cell = ds[D * 8 + e];
      if ((cell >= 0 && cell != x.s) || (x.s == prev_s && D * 8 + e != prev_cell)) { ok = false; break; }
      cell = x.s;
      prev_s = x.s, prev_cell = D * 8 + e;
      mask |= 1u << D;
    }
    if (!ok) continue;
    int64_t triples = 0, issued = 0;
    for (int D = 0; D < 27; ++D) {
      if (!((mask >> D) & 1u)) continue;
      const int Dv[3] = {D / 9 - 1, (D / 3) % 3 - 1, D % 3 - 1};
      for (int d = 0; d < 8; ++d)
        for (int e = 0; e < 8; ++e) {
          int inf = 0;
          for (int i = 0; i < 3; ++i)
            inf = std::max(inf, std::abs(2 * Dv[i] + ((e >> (2 - i)) & 1) - ((d >> (2 - i)) & 1)));
          ++issued;  // the kernel runs all 64 pairs (adjacent ones against zero tables)
          if (inf < 2) continue;
          if (dt[d] >= 0 && ds[D * 8 + e] >= 0) ++triples;
        }
    }
    if (triples != (int64_t)ents.size()) continue;
    macs += issued;
    return true;
  }
  return false;
}

static void upload_sym_table() {  // __constant__ memory is per device: upload once per device
  std::lock_guard<std::recursive_mutex> lk(cache_mutex());
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
  // parent-block form when every group has one and it does not waste too many MACs
  std::vector<int32_t> dtg((size_t)G * 8), dsr((size_t)G * 27 * 8);
  std::vector<uint32_t> dmk((size_t)G);
  bool dense = G > 0;
  int64_t macs = 0, entries = 0;
  for (int64_t g = 0; g < G && dense; ++g) {
    const int na = (int)(gb[g + 1] - gb[g]);
    int32_t tg[8];
    for (int a = 0; a < na; ++a) tg[a] = (int32_t)(gb[g] + a);
    entries += row[gb[g + 1]] - row[gb[g]];
    dense = dense_group(na, tg, row, src, oid, &dtg[(size_t)g * 8], &dsr[(size_t)g * 27 * 8], dmk[g], macs);
  }
  const char *force_list = getenv("HFMM_M2L_LIST");
  if (force_list && atoi(force_list) != 0) dense = false;
  if (dense && macs > 0 && (double)entries >= HFMM_M2L_DENSE_MIN * (double)macs) {
    pl->dense = true;
    pl->dense_macs = macs;
  }
  auto up = [](const void *h, size_t bytes) -> void * {
    void *d = nullptr;
    if (bytes && cudaMalloc(&d, bytes) == cudaSuccess) cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    return d;
  };
  pl->gtarget = (int32_t *)up(gt.data(), gt.size() * 4);
  pl->gsrc_row = (int32_t *)up(grow.data(), grow.size() * 4);
  pl->src_box = (int32_t *)up(sbox.data(), sbox.size() * 4);
  pl->tid8 = (int16_t *)up(t8.data(), t8.size() * 2);
  if (pl->dense) {
    pl->dtarget = (int32_t *)up(dtg.data(), dtg.size() * 4);
    pl->dsrc = (int32_t *)up(dsr.data(), dsr.size() * 4);
    pl->dmask = (uint32_t *)up(dmk.data(), dmk.size() * 4);
  }
  return pl;
}

int m2l_group_plan_kind(const M2LGroupPlan *pl) { return pl ? (pl->dense ? 1 : 0) : -1; }

void m2l_group_plan_destroy(M2LGroupPlan *pl) {
  if (!pl) return;
  for (void *p : {(void *)pl->gtarget, (void *)pl->gsrc_row, (void *)pl->src_box, (void *)pl->tid8,
                  (void *)pl->dtarget, (void *)pl->dsrc, (void *)pl->dmask})
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
  // units = (chunk, range of groups) in chunk-major order over persistent CTAs, so the CTAs
  // running at any time share about one chunk and its slice of M stays L2-resident.  A unit holds
  // whole groups per warp (1..4: balanced warps, the table fill amortised over up to 64 groups).
  const int64_t per_warp = std::max<int64_t>(1, std::min<int64_t>(4, pl->ngroups / ((int64_t)nsm * M2LG_WARPS)));
  const int64_t gpu = per_warp * M2LG_WARPS;
  const int64_t ranges = (pl->ngroups + gpu - 1) / gpu;
  const int64_t nunits = nchunks * ranges;
  const unsigned grid = (unsigned)std::min<int64_t>(nunits, nsm);
  if (pl->dense) {
    upload_slot_table();
    const size_t smem_b = (size_t)M2LB_SLOTS * M2LG_KC * sizeof(double2);
    cudaFuncSetAttribute(m2l_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    if (HFMM_M2L_PF16) {
      const size_t smem_p = ((size_t)M2LB_SLOTS * M2LP_KC + (size_t)M2LP_WARPS * 2 * 8 * 32) * sizeof(double2);
      cudaFuncSetAttribute(m2l_dense_pf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p);
      // units over 16-direction chunks: 16 warps x 2 groups cover groups_per_unit = per_warp x 32
      const int64_t nch16 = (pl->K + M2LP_KC - 1) / M2LP_KC;
      const int64_t gpu16 = per_warp * 2 * M2LP_WARPS;
      const int64_t ranges16 = (pl->ngroups + gpu16 - 1) / gpu16;
      const int64_t nunits16 = nch16 * ranges16;
      const unsigned grid16 = (unsigned)std::min<int64_t>(nunits16, nsm);
      m2l_dense_pf_kernel<<<grid16, 32 * M2LP_WARPS, smem_p, s>>>(pl->K, pl->ngroups, gpu16, nunits16, pl->dtarget,
                                                                  pl->dsrc, pl->dmask, T, perm, M, I);
    } else if (HFMM_M2L_GPW == 2) {
      cudaFuncSetAttribute(m2l_dense2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
      // same units (groups_per_unit = per_warp x 16): 8 warps x 2 groups each cover them
      m2l_dense2_kernel<<<grid, 32 * M2LB2_WARPS, smem_b, s>>>(pl->K, pl->ngroups, gpu, nunits, pl->dtarget,
                                                               pl->dsrc, pl->dmask, T, perm, M, I);
    } else if (HFMM_M2L_DMMA) {
      const size_t smem_d = ((size_t)M2LB_SLOTS * M2LD_KC + 2 * 64 * M2LD_MP) * sizeof(double2) + 8 * 27 * 8 * sizeof(int32_t);
      cudaFuncSetAttribute(m2l_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
      // units = (8-direction chunk, range of 8-group batches), chunk-major over persistent CTAs
      // (3 per SM); a unit holds up to 4 batches per CTA (the table fill amortised over 32 groups)
      const int64_t nch = (pl->K + M2LD_KC - 1) / M2LD_KC;
      const int64_t nbatch = (pl->ngroups + 7) / 8;
      const int64_t bpu = std::max<int64_t>(1, std::min<int64_t>(4, nbatch / (3 * (int64_t)nsm)));
      const int64_t rng = (nbatch + bpu - 1) / bpu;
      const int64_t nu = nch * rng;
      const unsigned gridd = (unsigned)std::min<int64_t>(nu, 3 * (int64_t)nsm);
      m2l_dmma_kernel<<<gridd, 32 * M2LD_WARPS, smem_d, s>>>(pl->K, pl->ngroups, bpu, nu, pl->dtarget, pl->dsrc,
                                                            pl->dmask, T, perm, M, I);
    } else {
      m2l_dense_kernel<<<grid, 32 * M2LG_WARPS, smem_b, s>>>(pl->K, pl->ngroups, gpu, nunits, pl->dtarget, pl->dsrc,
                                                           pl->dmask, T, perm, M, I);
    }
  } else {
    m2l_group_kernel<<<grid, 32 * M2LG_WARPS, smem, s>>>(pl->K, pl->ngroups, gpu, nunits, pl->gtarget,
                                                         pl->gsrc_row, pl->src_box, pl->tid8, T, perm, M, I);
  }
}

}  // namespace hfmm
