// Fused two-pass upward resampler (interpolation / M2M, P:119-122 with the 5-step procedure of
// P:738-748), product code, sm_100a.
//
// The register-resident passes of kernels_fft.cu (rows2 -> global intermediate -> cols2) move the
// intermediate (full parent-length rows n <= N_theta/2 of every child) through HBM: 1.8x the
// algorithmic bytes on the C2 B64 interpolation (profiles/r01).  Here ONE persistent kernel runs
// both passes as dependent tasks taken in a fixed order from a global counter:
//     round r:  the row task of every child of item r       (child -> ring slot r mod D)
//               the column task of item r - L              (ring slot -> parent, shift, child sum)
// A column task of item i waits for the row tasks of item i (per-item counter), a row task that
// reuses ring slot s waits until every column task of the item that last used it is done; both
// wait only on tasks with smaller positions in the order, which were handed out earlier to
// resident CTAs, so the waits always finish.  With the lag L and the ring of D items sized to a
// fraction of the 126 MB L2, the intermediate is produced and consumed in L2: HBM sees the
// algorithmic bytes (children read once, parents written once).
// Same arithmetic, operation for operation, as the two-pass kernels (the row / column task bodies
// are the rows2 / cols2 UP code), so results equal theirs bitwise (tests/test_gpu_fused.py).
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "hfmm_impl.h"
#include "fft_regs.cuh"

namespace hfmm {

constexpr int FU_CW = 8, FU_CWP = 9;   // columns per strip, exchange pitch (the cols2 layout)
#ifndef HFMM_FUSED_MINB
#define HFMM_FUSED_MINB 3                 // CTAs per SM asked of ptxas (the two-pass kernels run 3)
#endif

__device__ __forceinline__ void fu_cp_async16(double2 *smem, const double2 *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void fu_cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ int fu_ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
struct FuCfg {
  static constexpr int NR = RF1 * RF2, NR2 = RI1 * RI2;   // rows: N_phi -> N'_phi
  static constexpr int NC = CF1 * CF2, NC2 = CI1 * CI2;   // columns: N_theta -> N'_theta
  static constexpr int h = NR / 2, h2 = NR2 / 2, nrow = NC / 2 + 1;
  static constexpr int GM = Max2<Max2<RF1, RF2>::v, Max2<RI1, RI2>::v>::v;
  static constexpr int G = GM <= 1 ? 1 : GM <= 2 ? 2 : GM <= 4 ? 4 : GM <= 8 ? 8 : 16;
  static constexpr int VW = 32 / G;
  static constexpr int RBUF = Max2<Max2<RF1 * (RF2 + 1), RI1 * (RI2 + 1)>::v, Max2<NR, NR2>::v>::v;
  static constexpr int CBUF = Max2<Max2<CF1 * (CF2 + 1), CI1 * (CI2 + 1)>::v, Max2<NC, NC2>::v>::v;
  static constexpr int NSTRIP = (h2 + FU_CW - 1) / FU_CW;
  static constexpr size_t child_elems = (size_t)nrow * NR2;          // intermediate of one child
  static constexpr size_t row_smem = (size_t)4 * VW * RBUF;
  static constexpr size_t col_smem = (size_t)(CBUF + NC) * FU_CWP;
  static constexpr size_t smem_elems() {
    return (size_t)NR + NR2 + NC + NC2 + (row_smem > col_smem ? row_smem : col_smem);
  }
};

template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
__global__ void __launch_bounds__(128, HFMM_FUSED_MINB) fused_up_kernel(const double2 *__restrict__ in, int64_t nitem,
                                                      const int32_t *__restrict__ cbeg, int64_t cbase, int CH,
                                                      const int8_t *__restrict__ oct,
                                                      const double2 *__restrict__ shift,
                                                      const double2 *__restrict__ twR, const double2 *__restrict__ twR2,
                                                      const double2 *__restrict__ twC, const double2 *__restrict__ twC2,
                                                      double2 *__restrict__ out, double2 *__restrict__ ring,
                                                      int64_t D, int64_t L, int *__restrict__ rows_done,
                                                      int *__restrict__ cols_done, int *__restrict__ queue) {
  using C = FuCfg<RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  constexpr int NR = C::NR, NR2 = C::NR2, NC = C::NC, NC2 = C::NC2, h = C::h, h2 = C::h2, nrow = C::nrow;
  constexpr int G = C::G, VW = C::VW, RBUF = C::RBUF, CBUF = C::CBUF, NSTRIP = C::NSTRIP;
  constexpr int KR = ((NR < NR2 ? NR : NR2) - 1) / 2, KC = ((NC < NC2 ? NC : NC2) - 1) / 2;
  extern __shared__ double2 sm[];
  double2 *tr1 = sm, *tr2 = tr1 + NR, *tc1 = tr2 + NR2, *tc2 = tc1 + NC;
  double2 *work = tc2 + NC2;
  double2 *rbuf = work;                          // row tasks: [4 warps][VW][RBUF]
  double2 *cbuf = work, *stg = work + CBUF * FU_CWP;   // column tasks: exchange + staged strip
  __shared__ int64_t s_task;
  for (int j = threadIdx.x; j < NR; j += blockDim.x) tr1[j] = twR[j];
  for (int j = threadIdx.x; j < NR2; j += blockDim.x) tr2[j] = twR2[j];
  for (int j = threadIdx.x; j < NC; j += blockDim.x) tc1[j] = twC[j];
  for (int j = threadIdx.x; j < NC2; j += blockDim.x) tc2[j] = twC2[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, gr = lane - grp * G;
  double2 *rb = rbuf + (warp * VW + grp) * RBUF;
  const int v = threadIdx.x & (FU_CW - 1), g = threadIdx.x >> 3;
  const int64_t RT = CH + 1;                      // tasks per round: the row tasks, one column task
  const int64_t ntasks = (nitem + L) * RT;
  for (;;) {
    __syncthreads();                              // previous task done with shared memory / s_task
    if (threadIdx.x == 0) s_task = atomicAdd(queue, 1);
    __syncthreads();
    const int64_t t = s_task;
    if (t >= ntasks) break;
    const int64_t round = t / RT, idx = t - round * RT;
    if (idx < CH) {
      // ---------------- row task: child j of item `round` -> ring slot ----------------
      const int64_t item = round;
      if (item >= nitem) continue;
      const int64_t c0 = cbeg ? cbeg[item] : item, c1 = cbeg ? cbeg[item + 1] : item + 1;
      const int64_t c = c0 + idx;
      if (c >= c1) continue;
      if (item >= D) {                            // slot reuse: the item D before must be consumed
        if (threadIdx.x == 0)
          while (fu_ld_acquire(&cols_done[item - D]) < 1) __nanosleep(64);
        __syncthreads();
      }
      double2 *dst = ring + ((item % D) * CH + idx) * C::child_elems;
      const double2 *src = in + (c - cbase) * (int64_t)NC * h;
      for (int r0 = warp * VW; r0 < nrow; r0 += 4 * VW) {
        const int n = r0 + grp;
        const bool vok = n < nrow;
        double2 x[16];
        if (vok && gr < RF2) {
          const double2 *lo = src + (int64_t)n * h, *hi = src + (int64_t)(n == 0 ? 0 : NC - n) * h;
#pragma unroll
          for (int n1 = 0; n1 < RF1; ++n1) {
            const int e = RF2 * n1 + gr;
            x[n1] = e < h ? lo[e] : hi[e - h];
          }
          dft<RF1>(x);
#pragma unroll
          for (int k1 = 1; k1 < RF1; ++k1) x[k1] = c_mul(x[k1], tr1[gr * k1]);
#pragma unroll
          for (int k1 = 0; k1 < RF1; ++k1) rb[k1 * (RF2 + 1) + gr] = x[k1];
        }
        __syncwarp();
        if (vok && gr < RF1) {
#pragma unroll
          for (int n2 = 0; n2 < RF2; ++n2) x[n2] = rb[gr * (RF2 + 1) + n2];
        }
        __syncwarp();
        if (vok && gr < RF1) {
          dft<RF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < RF2; ++k2) rb[gr + RF1 * k2] = x[k2];
        }
        __syncwarp();
        if (vok && gr < RI2) {
#pragma unroll
          for (int m1 = 0; m1 < RI1; ++m1) {
            const int i = RI2 * m1 + gr;
            const int f = (i <= NR2 / 2) ? i : i - NR2;
            double2 z = make_double2(0.0, 0.0);
            if (f <= KR && f >= -KR) {
              const double2 y = rb[f >= 0 ? f : f + NR];
              z = make_double2(y.x * (1.0 / NR), -y.y * (1.0 / NR));
            }
            x[m1] = z;
          }
        }
        __syncwarp();
        if (vok && gr < RI2) {
          dft<RI1>(x);
#pragma unroll
          for (int k1 = 1; k1 < RI1; ++k1) x[k1] = c_mul(x[k1], tr2[gr * k1]);
#pragma unroll
          for (int k1 = 0; k1 < RI1; ++k1) rb[k1 * (RI2 + 1) + gr] = x[k1];
        }
        __syncwarp();
        if (vok && gr < RI1) {
#pragma unroll
          for (int n2 = 0; n2 < RI2; ++n2) x[n2] = rb[gr * (RI2 + 1) + n2];
          dft<RI2>(x);
          double2 *o = dst + (int64_t)n * NR2;
#pragma unroll
          for (int k2 = 0; k2 < RI2; ++k2) o[gr + RI1 * k2] = c_conj(x[k2]);
        }
        __syncwarp();
      }
      __threadfence();                            // the slot's rows visible GPU-wide ...
      __syncthreads();
      if (threadIdx.x == 0) atomicAdd(&rows_done[item], 1);   // ... before the count
    } else {
      // ------- column task: every strip of item `round - L` (ring -> parent), the next step's
      //         strip fetched with cp.async while the current one is transformed (cols2 pipeline)
      const int64_t item = round - L;
      if (item < 0 || item >= nitem) continue;
      const int64_t c0 = cbeg ? cbeg[item] : item, c1 = cbeg ? cbeg[item + 1] : item + 1;
      const int nch = (int)(c1 - c0);
      if (threadIdx.x == 0)
        while (fu_ld_acquire(&rows_done[item]) < nch) __nanosleep(64);
      __syncthreads();
      const double2 *slot = ring + (item % D) * CH * C::child_elems;
      auto issue = [&](int st) {   // step st = strip * nch + child
        const int strip = st / nch, cj = st - strip * nch;
        const double2 *cb = slot + cj * C::child_elems;
        for (int e = threadIdx.x; e < NC * FU_CW; e += blockDim.x) {   // theta-periodic strip (L2 only)
          const int n = e >> 3, vv = e & (FU_CW - 1), mm = strip * FU_CW + vv;
          if (mm >= h2) continue;
          const double2 *sp = (2 * n <= NC) ? &cb[(int64_t)n * NR2 + mm] : &cb[(int64_t)(NC - n) * NR2 + mm + h2];
          fu_cp_async16(&stg[n * FU_CWP + vv], sp);
        }
      };
      const int nsteps = NSTRIP * nch;
      issue(0);
      for (int st = 0; st < nsteps; ++st) {
        const int strip = st / nch, cj = st - strip * nch;
        const int64_t c = c0 + cj;
        const int m = strip * FU_CW + v;
        const bool mok = m < h2;
        double2 *ob = out + item * (int64_t)NC2 * h2 + m;
        double2 x[16];
        fu_cp_async_wait_all();
        __syncthreads();                          // stg holds step st; cbuf free
        if (g < CF2) {
#pragma unroll
          for (int n1 = 0; n1 < CF1; ++n1) x[n1] = mok ? stg[(CF2 * n1 + g) * FU_CWP + v] : make_double2(0.0, 0.0);
          dft<CF1>(x);
#pragma unroll
          for (int k1 = 1; k1 < CF1; ++k1) x[k1] = c_mul(x[k1], tc1[g * k1]);
#pragma unroll
          for (int k1 = 0; k1 < CF1; ++k1) cbuf[(k1 * (CF2 + 1) + g) * FU_CWP + v] = x[k1];
        }
        __syncthreads();                          // stg consumed: fetch the next step's strip
        if (st + 1 < nsteps) issue(st + 1);
        if (g < CF1) {
#pragma unroll
          for (int n2 = 0; n2 < CF2; ++n2) x[n2] = cbuf[(g * (CF2 + 1) + n2) * FU_CWP + v];
        }
        __syncthreads();
        if (g < CF1) {
          dft<CF2>(x);
#pragma unroll
          for (int k2 = 0; k2 < CF2; ++k2) cbuf[(g + CF1 * k2) * FU_CWP + v] = x[k2];
        }
        __syncthreads();
        if (g < CI2) {
#pragma unroll
          for (int m1 = 0; m1 < CI1; ++m1) {
            const int i = CI2 * m1 + g;
            const int f = (i <= NC2 / 2) ? i : i - NC2;
            double2 z = make_double2(0.0, 0.0);
            if (f <= KC && f >= -KC) {
              const double2 y = cbuf[(f >= 0 ? f : f + NC) * FU_CWP + v];
              z = make_double2(y.x * (1.0 / NC), -y.y * (1.0 / NC));
            }
            x[m1] = z;
          }
        }
        __syncthreads();
        if (g < CI2) {
          dft<CI1>(x);
#pragma unroll
          for (int k1 = 1; k1 < CI1; ++k1) x[k1] = c_mul(x[k1], tc2[g * k1]);
#pragma unroll
          for (int k1 = 0; k1 < CI1; ++k1) cbuf[(k1 * (CI2 + 1) + g) * FU_CWP + v] = x[k1];
        }
        __syncthreads();
        if (g < CI1 && mok) {
#pragma unroll
          for (int n2 = 0; n2 < CI2; ++n2) x[n2] = cbuf[(g * (CI2 + 1) + n2) * FU_CWP + v];
          dft<CI2>(x);
#pragma unroll
          for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_conj(x[k2]);
          if (shift) {
            const double2 *sb = shift + (int64_t)(oct ? oct[c] : 0) * NC2 * h2 + m;
            double2 tt[CI2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) tt[k2] = __ldg(&sb[(int64_t)(g + CI1 * k2) * h2]);
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_mul(x[k2], tt[k2]);
          }
          if (cj != 0) {
            double2 tt[CI2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) tt[k2] = ob[(int64_t)(g + CI1 * k2) * h2];
#pragma unroll
            for (int k2 = 0; k2 < CI2; ++k2) x[k2] = c_add(x[k2], tt[k2]);
          }
#pragma unroll
          for (int k2 = 0; k2 < CI2; ++k2) ob[(int64_t)(g + CI1 * k2) * h2] = x[k2];
        }
      }
      __syncthreads();                            // every thread's ring reads done
      if (threadIdx.x == 0) atomicAdd(&cols_done[item], 1);
    }
  }
}

// ---- launch ---------------------------------------------------------------------------------------
// Process-wide switch: HFMM_FUSED in the environment at load time (default 0), or hfmm_set_fused().
// Off by default: the same-box A/B lost (profiles/r02/fused_ab_r2.txt: B64 interp 27.5 / 21.7 ms
// at 3 / 2 CTAs per SM vs 17.1 ms two-pass; fused M2M far slower -- one column task per parent
// serialises 8 children x 16 strips behind the dependency waits).  The two-pass kernels run at
// ~4.5 TB/s average on their 1.8x traffic; the task-queue kernel is latency-bound instead.
static std::atomic<int> g_fused{[] {
  const char *e = getenv("HFMM_FUSED");
  return e ? atoi(e) : 0;
}()};

bool fused_enabled() { return g_fused.load(std::memory_order_relaxed) != 0; }

}  // namespace hfmm

extern "C" int hfmm_set_fused(int on) { return hfmm::g_fused.exchange(on ? 1 : 0); }

namespace hfmm {

// ring: caller's workspace (ring_elems complex values); cnt: caller's 2 nitem + 1 ints (zeroed here)
template <int RF1, int RF2, int RI1, int RI2, int CF1, int CF2, int CI1, int CI2>
static bool launch_fused_up_t(const double2 *in, int64_t nitem, const int32_t *cbeg, int64_t cbase, const int8_t *oct,
                              const double2 *shift, double2 *out, double2 *ring, size_t ring_elems, int *cnt,
                              const TwiddleSet &tw, cudaStream_t s) {
  using C = FuCfg<RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  const int CH = cbeg ? 8 : 1;
  const size_t item_elems = (size_t)CH * C::child_elems;
  // ring of D items within ~64 MB of the 126 MB L2 (the rest holds the streaming data), lag L = D/2
  int64_t D = (int64_t)((64ull << 20) / (item_elems * sizeof(double2)));
  D = std::min<int64_t>({D, (int64_t)(ring_elems / item_elems), std::max<int64_t>(nitem, 1)});
  if (D < 2 || !cnt) return false;
  const int64_t L = std::max<int64_t>(1, D / 2);
  cudaMemsetAsync(cnt, 0, (2 * nitem + 1) * sizeof(int), s);
  const size_t smem = C::smem_elems() * sizeof(double2);
  auto kern = fused_up_kernel<RF1, RF2, RI1, RI2, CF1, CF2, CI1, CI2>;
  cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
  // persistent CTAs; tasks are claimed only by running CTAs, so the waits need no co-residency
  const unsigned grid = (unsigned)std::max(1, nsm * std::max(per, 1));
  kern<<<grid, 128, smem, s>>>(in, nitem, cbeg, cbase, CH, oct, shift, tw.d + tw.offset[C::NR],
                               tw.d + tw.offset[C::NR2], tw.d + tw.offset[C::NC], tw.d + tw.offset[C::NC2], out, ring, D,
                               L, cnt, cnt + nitem, cnt + 2 * nitem);
  return true;
}

// (nth, nph) -> (nth2, nph2) with a fused kernel: the large square grids of the C2 microbench
bool launch_fused_up(const double2 *in, int64_t nitem, int nth, int nph, int nth2, int nph2, const int32_t *cbeg,
                     int64_t cbase, const int8_t *oct, const double2 *shift, double2 *out, double2 *ring,
                     size_t ring_elems, int *cnt, const TwiddleSet &tw, cudaStream_t s) {
  if (!fused_enabled()) return false;
  const int64_t key = ((((int64_t)nth * 1000 + nph) * 1000 + nth2) * 1000 + nph2);
  switch (key) {
    case ((((int64_t)64 * 1000 + 64) * 1000 + 128) * 1000 + 128):
      return launch_fused_up_t<8, 8, 16, 8, 8, 8, 16, 8>(in, nitem, cbeg, cbase, oct, shift, out, ring, ring_elems, cnt,
                                                                           tw, s);
    case ((((int64_t)128 * 1000 + 128) * 1000 + 256) * 1000 + 256):
      return launch_fused_up_t<16, 8, 16, 16, 16, 8, 16, 16>(in, nitem, cbeg, cbase, oct, shift, out, ring, ring_elems, cnt,
                                                                           tw, s);
    default: return false;
  }
}

}  // namespace hfmm
