/*
 * hfmm.h -- C ABI of libhfmm, a B200 (sm_100a) implementation of the Fourier-basis
 * Helmholtz fast multipole matrix-vector product of Cecka & Darve (arXiv 0911.4114).
 *
 * Citations "P:n" are line numbers of /root/reference/PAPER.md (the paper's LaTeX source).
 *
 * The operation (eqn:HelmholtzMatrixVector):
 *
 *     y_i = sum_{j != i} exp(i kappa |x_i - x_j|) / |x_i - x_j| * q_j ,   i = 0..n-1
 *
 * (no 1/(4 pi) factor; the self term is excluded), evaluated by the FMM of P:114-138:
 * S2M at the far-field leaf level, M2M with FFT interpolation,
 * diagonal M2L with the bandlimited modified transfer function of Alg. 1 (P:123-127,
 * P:508-530), L2L with FFT anterpolation, L2T + P2P near field
 * (eqn:FMM_FinalStep).
 *
 * Conventions
 *   - complex numbers are interleaved float64 pairs (re, im), i.e. C99 double _Complex /
 *     numpy complex128 / torch.complex128 memory layout;
 *   - positions are row-major n x 3 float64 (x0 y0 z0 x1 y1 z1 ...);
 *   - every array argument is owned by the caller; the library copies what it keeps;
 *   - a plan is NOT thread-safe; distinct plans are independent;
 *   - state machine: create -> build_tree -> precompute -> matvec*; build_tree again
 *     invalidates the precompute (HFMM_E_STATE if matvec is called too early);
 *   - return value: 0 success, > 0 warning (result still valid), < 0 error; the message
 *     of the last non-zero return is available from hfmm_last_error(plan).
 *
 * Multi-GPU: call hfmm_set_dist() between create and build_tree; every rank then calls
 * every function collectively with identical arguments (inputs replicated).  Each rank
 * computes the far field and near field of the level-2 subtrees it owns (Morton-ordered
 * partition weighted by work); multipole expansions of every active level are
 * all-gathered with NCCL over NVLink before M2L; y is all-gathered at the end (each rank's
 * owned sorted range, then unpermuted on every rank) unless HFMM_Y_LOCAL is set (then only owned
 * entries of y are written, others are zero).
 */
#ifndef HFMM_H
#define HFMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes -------------------------------------------------------------------- */
#define HFMM_OK 0
#define HFMM_W_BREAKDOWN 1    /* some levels inadmissible (L_f < depth)            */
#define HFMM_W_NO_FARFIELD 2  /* no admissible level: the matvec is the direct sum         */
#define HFMM_E_ARG (-1)       /* bad argument: n <= 0, depth < 2, kappa <= 0, eps not in
                                 (0,1), alpha not in (0,1], non-finite input, NULL pointer */
#define HFMM_E_DOMAIN (-2)    /* a point lies outside the root cube                         */
#define HFMM_E_COINCIDENT (-3) /* two distinct points coincide (kernel undefined at R = 0) */
#define HFMM_E_SEARCH (-4)    /* no ell / N_theta / N_phi within the search limits (Algs 2-3)*/
#define HFMM_E_STATE (-5)     /* call out of order                                          */
#define HFMM_E_NOMEM (-6)     /* device or host allocation failed                           */
#define HFMM_E_CUDA (-7)      /* CUDA runtime error (message has the CUDA error string)     */
#define HFMM_E_NCCL (-8)      /* NCCL error                                                 */

/* ---- precompute flags ---------------------------------------------------------------- */
#define HFMM_EPS_ABSOLUTE 0x1u     /* use eps itself at every level (default eps/a_l)        */
#define HFMM_FORCE_ALL_LEVELS 0x2u /* run M2L at every level 2..depth regardless of F_l
                                      (low-frequency breakdown demonstration)        */
#define HFMM_ALPHA_FIXED 0x4u      /* use the caller's alpha at every level (the paper's fixed
                                      design radius); default: per level the largest alpha in
                                      {1, 0.9, 0.8} (>= the caller's) that keeps F_l <= tau   */
#define HFMM_SOURCE_AT_LF 0x8u     /* S2M / L2T at L_f (the paper's setup, no translation-only
                                      levels); default: source level D_s by the policy below */
#define HFMM_RAGGED 0x20u          /* ragged quadrature on the active levels (R-15, Alg. 3 per row;
                                      SURVEY 8f NEXT 2); default: rectangular N_phi (R-4)    */
#define HFMM_DETERMINISTIC 0x40u   /* bitwise-reproducible near field (the DEFAULT; kept as an explicit
                                      request): every P2P work item writes its row / column partial
                                      sums to its own slots (no atomics) and each point sums its
                                      partials in a fixed order -- C4: +0.2% time, ~1.5 GB of
                                      partials and indices (C5: ~20 GB)                        */
#define HFMM_ATOMIC_NEAR 0x80u     /* opt out of the above: P2P partial sums added with atomics
                                      (no partial buffers; repeat runs agree to ~1e-16 only)   */
#define HFMM_SOURCE_AT_DEPTH 0x10u /* S2M / L2T at the configured depth D.  Default policy
                                      (R-14): the deepest level <= D whose occupied
                                      boxes hold >= 8 points on average; levels L_f < l <= D_s
                                      are translation-only (M2M up / L2L down, no M2L)
                                      on grids whose dropped Jacobi-Anger tail of
                                      eqn:PlaneWaveSpec is <= eps / 100        */

/* ---- matvec memory kinds -------------------------------------------------------------- */
#define HFMM_HOST 0    /* q and y are host pointers (pinned or pageable)                     */
#define HFMM_DEVICE 1  /* q and y are device pointers on the plan's device                   */
#define HFMM_Y_LOCAL 2 /* OR-able with the above: multi-GPU, skip the final y all-gather     */
#define HFMM_SERIAL 4  /* OR-able: near field and far chain one after the other on one stream
                          (measurement: kernel times without the two streams sharing SMs)   */

#define HFMM_MAX_LEVELS 16

typedef struct hfmm_plan hfmm_plan; /* opaque; owns all device memory and the NCCL comm */

typedef struct {
  int level;        /* l (box size a_l = a_0 / 2^l)                                  */
  double a;         /* a_l                                                                 */
  int ell;          /* Gegenbauer truncation                                   */
  int n_theta;      /* N_theta (Alg. 2), even, 7-smooth                         */
  int n_phi;        /* N_phi (Alg. 3), multiple of 4, 7-smooth                  */
  double alpha;     /* design radius |r| = alpha sqrt(3) a_l used for this level   */
  int64_t K;        /* stored quadrature points N_theta * N_phi / 2            */
  double F;         /* roundoff amplification 8 pi u a_l max|T_l| (NaN if not evaluated)    */
  int active;       /* 1 if M2L runs at this level                                         */
  int64_t boxes;    /* occupied boxes at this level                                        */
  int64_t m2l_pairs;/* interaction-list entries at this level (all ranks)                  */
  int rep;          /* 1: translation-only level L_f < l <= D_s (R-14; ell = 0, F = NaN)   */
  int ragged;       /* 1: ragged rows N_phi(theta_n) (R-15, HFMM_RAGGED); K = stored points   */
  int m2l_block;    /* 1: M2L runs the parent-block kernel, 0: the merged-list kernel (both
                       compute exactly the interaction-list sum; M2L)             */
  int halo;         /* multi-rank: 1 if M_l is exchanged as M2L halos (grouped ncclSend /
                       ncclRecv of the peers' boxes in this rank's interaction lists; levels
                       >= HFMM_HALO_LEVEL, default 4), 0 if all-gathered                      */
  int64_t m_recv_boxes; /* multi-rank: boxes of M_l this rank receives per matvec (0: one rank) */
  int64_t m_send_boxes; /* multi-rank: boxes of M_l this rank sends per matvec (sum over peers)  */
} hfmm_level_info;

typedef struct {
  int64_t n;               /* points                                                       */
  int depth;               /* configured depth D                                           */
  int L_f;                 /* far-field leaf level, or -1 if no admissible level             */
  double kappa, eps, alpha, tau;
  int nlevels;             /* entries filled in level[] (levels 2..D)                        */
  hfmm_level_info level[HFMM_MAX_LEVELS];
  int64_t p2p_pairs;       /* ordered near-field pairs i != j (owned targets)                */
  int64_t p2p_sym_pairs;   /* unordered pairs of them evaluated once (symmetric kernel)      */
  int64_t s2m_evals;       /* owned points x directions at the source level D_s             */
  int rank, nranks;
  int64_t owned_points;    /* points whose y this rank computes                              */
  int source_level;        /* D_s: level of S2M / L2T (R-14), -1 if no far field             */
  int launches;            /* libhfmm kernel launches per matvec (this rank)                 */
  int p2p_tile;            /* targets per P2P work item (128 threads x 3 or 4 targets each: 4
                              unless the items would fill fewer than ~10 waves of the GPU)     */
  int next4_passes;        /* M2M / L2L level passes run by the NEXT 4 coefficient-domain
                              symmetric kernels (HFMM_NEXT4=1 in the environment), else 0     */
  int p2p_rowskip;         /* 1: the symmetric P2P kernel skips 32-target warp rows wholly past
                              a tile's end (chosen when > 8% of the tile slots are dead)        */
  double p2p_dead_frac;    /* fraction of the P2P tile slots (128 x targets-per-thread x padded
                              sources) that hold no live target                                */
  int64_t p2p_mixed_items; /* mixed tiles: work items of the <= 384-point target-tile class (each
                              leaf cut into full 512-point tiles plus <= 384-point ones, one
                              launch per class); 0 when the plan uses one tile size             */
} hfmm_info;

/* Create a plan on CUDA device `device` (-1: the current device).  *out receives the plan. */
int hfmm_create(hfmm_plan **out, int device);

/* Multi-GPU: rank / nranks and the 128-byte ncclUniqueId (broadcast by the caller, e.g. with
 * torch.distributed).  nranks == 1 (default) disables all collectives. */
int hfmm_set_dist(hfmm_plan *p, int rank, int nranks, const void *nccl_unique_id_128b);

/* Fill out_128b with a fresh ncclUniqueId (rank 0 calls this and broadcasts the bytes). */
int hfmm_nccl_unique_id(void *out_128b);

/* Virtual ranks (test mode for the multi-rank path on ONE device, one process): a group of
 * nranks plans, each bound to a rank with hfmm_set_dist_virtual (instead of hfmm_set_dist,
 * before build_tree; every plan on the same device, built with identical arguments).  The
 * plans then partition the work exactly as nranks GPUs would.  hfmm_vgroup_matvec runs the
 * multi-rank matvec over all of them, every collective replaced by one cudaMemcpyAsync per peer
 * block (M_l all-gather before M2L, y all-gather at the end): q DEVICE pointer [n] complex128
 * (input order), y DEVICE pointer [nranks][n] (rank r's full output vector at y + r n); enqueued
 * on `stream` (NULL: rank 0's plan stream, synchronised before return).  A plan bound to a group
 * returns HFMM_E_STATE from hfmm_matvec.  Destroy the group after (or before) its plans. */
/* NEXT 4 (coefficient-domain symmetric resampling, eqn:FourierSphereSym P:277-280):
 * process-wide switch for the single-pass M2M / L2L / resample kernels of the grid pairs it is
 * instantiated for (C2 B8-B32, the translation-only levels of C3 / C4 / C5); other pairs keep the
 * 5-step kernels.  Initial value from HFMM_NEXT4 in the environment (default 0).  Set it before
 * hfmm_precompute (hfmm_info.next4_passes / launches are counted there).  Returns the previous
 * value. */
int hfmm_set_next4(int on);

/* Fused two-pass upward resampler (interpolation / M2M on the large grids: C2 B32 / B64): rows and
 * columns as dependent tasks of one persistent kernel with the intermediate in an L2-sized ring
 * (csrc/kernels_fused.cu).  Process-wide switch, default OFF (slower in the same-box A/B,
 * profiles/r02/fused_ab_r2.txt); HFMM_FUSED=1 in the environment turns it on at load; off = the
 * two-pass kernels with a global intermediate.  Returns the previous value. */
int hfmm_set_fused(int on);

typedef struct hfmm_vgroup hfmm_vgroup;
int hfmm_vgroup_create(hfmm_vgroup **out, int nranks);
int hfmm_set_dist_virtual(hfmm_plan *p, hfmm_vgroup *g, int rank);
int hfmm_vgroup_matvec(hfmm_vgroup *g, const double *q, double *y, void *stream);
void hfmm_vgroup_destroy(hfmm_vgroup *g);

/* Octree over n points.  xyz: HOST pointer, n x 3 row-major float64.  depth >= 2 is the
 * configured leaf level D (root level 0); root cube [lo, lo + size]^3 must contain every point
 * (HFMM_E_DOMAIN otherwise).  Box coordinate b = min(floor((x - lo) / a_l), 2^l - 1).
 * Detects exactly coincident points (HFMM_E_COINCIDENT).  Copies xyz to the device. */
int hfmm_build_tree(hfmm_plan *p, int64_t n, const double *xyz, int depth,
                    const double lo[3], double size);

/* Plan for wavenumber kappa > 0 and target accuracy eps in (0,1): per level ell (EBF +
 * Carayol-Collino), N_theta (Alg. 2), N_phi (Alg. 3), the 316 bandlimited modified
 * transfer tables (Alg. 1, computed on the GPU), F_l and the far-field leaf level L_f (deepest
 * level with F_2..F_l <= tau).  alpha in (0,1] scales the design radius |r| = alpha sqrt(3) a_l
 * (0.8 in the paper's error studies).  tau <= 0 selects min(eps/10, 1e-9).
 * Returns HFMM_W_BREAKDOWN / HFMM_W_NO_FARFIELD as warnings. */
int hfmm_precompute(hfmm_plan *p, double kappa, double eps, double alpha, double tau,
                    unsigned flags);

/* y = A q (eqn:HelmholtzMatrixVector).  q: n complex128 in INPUT order, y: n complex128 in
 * input order.  mem = HFMM_HOST or HFMM_DEVICE (optionally | HFMM_Y_LOCAL).  stream: a
 * cudaStream_t on the plan's device (cudaStreamLegacy = (void*)1 for the legacy default
 * stream), or NULL for the plan's own stream.  The call returns after y is written for
 * HFMM_HOST and for a NULL stream; for HFMM_DEVICE with an explicit stream it returns after
 * enqueueing (y valid once `stream` reaches that point).  Input q is read, and y written, in
 * stream order on `stream`. */
int hfmm_matvec(hfmm_plan *p, const double *q, double *y, int mem, void *stream);

/* Direct O(n^2) sum on the GPU (same P2P kernel over all pairs), same conventions. */
int hfmm_direct(hfmm_plan *p, const double *q, double *y, int mem, void *stream);

/* Plan summary (valid after precompute). */
int hfmm_get_info(const hfmm_plan *p, hfmm_info *info);

/* Device timing of the stages of the last matvec in milliseconds (CUDA events on the
 * launching streams): out[0] S2M, [1] M2M, [2] M2L, [3] L2L, [4] L2T, [5] P2P, [6] total.
 * Only filled when HFMM_PROFILE_STAGES is set in the environment. */
int hfmm_stage_times(const hfmm_plan *p, double out[8]);

/* Copy a stage buffer of the last matvec to host memory (testing and validation).
 * what: 0 M_l, 1 I_l (incoming), 2 L_l (local), 3 T_l (transfer tables [316][K_l]),
 *       4 y_near (sorted order), 5 y_far (sorted order), 6 permutation (int64, sorted -> input),
 *       7 box table of level l (int64 [boxes][4]: ix, iy, iz, first point),
 * level: tree level l.  nbytes: capacity of host_out.  Returns the bytes needed in *needed. */
int hfmm_debug_copy(const hfmm_plan *p, int what, int level, void *host_out, int64_t nbytes,
                    int64_t *needed);

/* Message of the last non-zero return of any call on p (or of hfmm_create if p is NULL). */
const char *hfmm_last_error(const hfmm_plan *p);

/* Free everything owned by the plan, including the NCCL communicator. */
void hfmm_destroy(hfmm_plan *p);

/* Host-only (no GPU needed): ragged rows of an active level (R-15; Alg. 3 per row,
 * P:669-684): rows[n], n < n_theta, = the smallest 7-smooth multiple of 4 at which row n passes
 * Alg. 3's test for (kappa, box size a, absolute level target eps_level, design radius alpha,
 * ell) at this n_theta, capped at n_phi_cap; rows n > n_theta/2 mirror n_theta - n.  Returns 0,
 * HFMM_E_ARG or HFMM_E_SEARCH. */
int hfmm_ragged_rows(double kappa, double a, double eps_level, double alpha, int ell, int n_theta,
                     int n_phi_cap, int *rows);

/* Host-only (no GPU needed): grid (N_theta, N_phi) of a translation-only level of box size a
 * (R-14; eqn:PlaneWaveSpec): smallest even 7-smooth N_theta >= 4 and
 * smallest 7-smooth multiple of 4 N_phi whose dropped Jacobi-Anger tail
 * 2 sum_{n >= N/2} |J_n(kappa (sqrt3/2) a)| is <= eps / 100.  Returns 0, HFMM_E_ARG or
 * HFMM_E_SEARCH. */
int hfmm_rep_grid(double kappa, double a, double eps, int *n_theta, int *n_phi);

/* ---- host-only plan helpers (no GPU needed) ---------------------------------------------
 * The per-level quadrature of P:140-722 for box size a: returns ell, N_theta, N_phi
 * (rectangular, 7-smooth) and fills ragged[0..N_theta/2] with Alg. 3's per-row N_phi(theta_n)
 * when ragged != NULL (capacity ragged_cap).  eps is the level's absolute target. */
int hfmm_level_quadrature(double kappa, double a, double eps_level, double alpha, int *ell,
                          int *n_theta, int *n_phi, int *ragged, int ragged_cap);

/* Host-only multi-GPU ownership (the rule hfmm_precompute applies; no GPU needed): for the tree
 * of (n, xyz, depth, lo, size), far-field leaf level L_f >= 2 and leaf quadrature size K, fills
 * cuts[0..nranks] (rank r owns level-2 boxes [cuts[r], cuts[r+1]) in Morton order, i.e. whole
 * subtrees), pt_ranges[2r], pt_ranges[2r+1] (its sorted-point range) and, if perm != NULL,
 * perm[0..n) (sorted position -> input index). */
int hfmm_partition(int64_t n, const double *xyz, int depth, const double lo[3], double size, int L_f,
                   int64_t K, int nranks, int64_t *cuts, int64_t *pt_ranges, int64_t *perm);

/* Host-only M2L halo lists (the exchange hfmm_precompute sets up for levels >= HFMM_HALO_LEVEL of
 * a multi-rank plan; no GPU needed): with the ownership of hfmm_partition(..., L_f, K, nranks, ...)
 * descended to `level` (2 <= level <= L_f), rank `rank` receives from each peer q the q-owned
 * level-`level` boxes in the interaction lists of its own boxes, and sends each peer q its
 * own boxes in the interaction lists of q's boxes.  Box ids index the occupied boxes of the level
 * in Morton order.  recv_off / send_off [nranks + 1] (always written): list of peer q =
 * [off[q], off[q+1]); recv_box / send_box: NULL (sizes only) or arrays of off[nranks] entries,
 * each list sorted ascending (so q's send list to r equals r's receive list from q).  Caller owns
 * all arrays.  Returns 0, or HFMM_E_ARG / a build_tree error. */
int hfmm_halo_lists(int64_t n, const double *xyz, int depth, const double lo[3], double size, int L_f,
                    int64_t K, int nranks, int rank, int level, int64_t *recv_off, int64_t *send_off,
                    int64_t *recv_box, int64_t *send_box);

/* ---- operator entry points (microbench, BASELINE config 2; device pointers) -----------------
 * Batched 5-step Fourier resampling of `nbatch` half-stored fields
 * [n_theta][n_phi/2] -> [n_theta2][n_phi2/2]: interpolation if the target grid
 * is larger, anterpolation if smaller.  in/out: device complex128.  work: device scratch of
 * hfmm_resample_workspace() bytes (NULL: allocated internally per call). */
int64_t hfmm_resample_workspace(int nbatch, int n_theta, int n_phi, int n_theta2, int n_phi2);
int hfmm_resample(int nbatch, int n_theta, int n_phi, int n_theta2, int n_phi2, const double *in,
                  double *out, void *work, void *stream);

/* Fused M2M of 8 children per parent (interpolate, multiply by shift[octant][K_parent],
 * accumulate): children [nparent*8][K_child] -> parents [nparent][K_parent]. */
int hfmm_m2m_op(int nparent, int n_theta, int n_phi, int n_theta2, int n_phi2, const double *child,
                const double *shift, double *parent, void *work, void *stream);

/* Fused L2L: child_out[c] = anterp(conj(shift[c % 8]) * parent[c / 8]) + incoming[c]. */
int hfmm_l2l_op(int nparent, int n_theta, int n_phi, int n_theta2, int n_phi2,
                const double *parent, const double *shift, const double *incoming,
                double *child_out, void *work, void *stream);

/* Diagonal M2L over a CSR interaction list: out[a][k] = sum_e T[oid[e]][k] * M[src[e]][k]
 * for e in [row[a], row[a+1]).  row: int32 [nbox+1], src: int32, oid: int32 (0..315); T [316][K],
 * M / out [nbox][K] complex128.  hfmm_m2l_op: DEVICE CSR, one-shot (copies the CSR to the host and
 * builds the sibling-group plan every call; synchronises `stream`).  For repeated application:
 * hfmm_m2l_op_plan (HOST CSR; consecutive boxes 8 at a time form a group -- siblings when boxes
 * are in Morton order; returns HFMM_E_ARG for an out-of-range src / oid), hfmm_m2l_op_apply
 * (device T / M / out, enqueued on `stream`), hfmm_m2l_op_free. */
int hfmm_m2l_op(int nbox, int64_t K, const int *row, const int *src, const int *oid,
                const double *T, const double *M, double *out, void *stream);
int hfmm_m2l_op_plan(int nbox, int64_t K, const int *row, const int *src, const int *oid, void **plan);
int hfmm_m2l_op_apply(const void *plan, const double *T, const double *M, double *out, void *stream);
void hfmm_m2l_op_free(void *plan);
/* Kernel a plan runs: 1 parent-block (every group of 8 is the children of one parent and its lists
 * are exactly the admissible children of the 26 neighbour parents -- proven per group at plan
 * time), 0 merged-list; -1 for NULL.  Setting HFMM_M2L_LIST=1 in the environment before a plan is
 * made forces the merged-list kernel (A/B testing). */
int hfmm_m2l_op_kind(const void *plan);

#ifdef __cplusplus
}
#endif
#endif /* HFMM_H */
