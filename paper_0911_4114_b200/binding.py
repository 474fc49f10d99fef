"""Thin ctypes binding of libhfmm (include/hfmm.h): argument marshalling only.

Every step of the matvec runs in libhfmm's CUDA kernels; this module never computes any
part of the method.  There is no CPU fallback: if libhfmm.so is missing or no GPU is
present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HFMM_LIB: an alternative in-tree build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("HFMM_LIB") or os.path.join(_HERE, "libhfmm.so")

HFMM_OK = 0
HFMM_W_BREAKDOWN = 1
HFMM_W_NO_FARFIELD = 2
HFMM_EPS_ABSOLUTE = 0x1
HFMM_FORCE_ALL_LEVELS = 0x2
HFMM_ALPHA_FIXED = 0x4
HFMM_SOURCE_AT_LF = 0x8
HFMM_SOURCE_AT_DEPTH = 0x10
HFMM_RAGGED = 0x20
HFMM_DETERMINISTIC = 0x40
HFMM_ATOMIC_NEAR = 0x80
HFMM_HOST = 0
HFMM_DEVICE = 1
HFMM_Y_LOCAL = 2
HFMM_SERIAL = 4
MAX_LEVELS = 16

EXPORTED = [
    "hfmm_create", "hfmm_set_dist", "hfmm_nccl_unique_id", "hfmm_build_tree", "hfmm_precompute", "hfmm_matvec",
    "hfmm_direct", "hfmm_get_info", "hfmm_stage_times", "hfmm_debug_copy", "hfmm_last_error",
    "hfmm_destroy", "hfmm_level_quadrature", "hfmm_resample_workspace", "hfmm_resample",
    "hfmm_m2m_op", "hfmm_l2l_op", "hfmm_m2l_op", "hfmm_partition", "hfmm_halo_lists", "hfmm_rep_grid",
    "hfmm_m2l_op_plan", "hfmm_m2l_op_apply", "hfmm_m2l_op_free", "hfmm_m2l_op_kind", "hfmm_ragged_rows",
    "hfmm_vgroup_create", "hfmm_set_dist_virtual", "hfmm_vgroup_matvec", "hfmm_vgroup_destroy",
    "hfmm_set_next4", "hfmm_set_fused",
]


class LevelInfo(C.Structure):
    _fields_ = [("level", C.c_int), ("a", C.c_double), ("ell", C.c_int), ("n_theta", C.c_int),
                ("n_phi", C.c_int), ("alpha", C.c_double), ("K", C.c_int64), ("F", C.c_double),
                ("active", C.c_int),
                ("boxes", C.c_int64), ("m2l_pairs", C.c_int64), ("rep", C.c_int), ("ragged", C.c_int),
                ("m2l_block", C.c_int), ("halo", C.c_int), ("m_recv_boxes", C.c_int64),
                ("m_send_boxes", C.c_int64)]


class Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("depth", C.c_int), ("L_f", C.c_int), ("kappa", C.c_double),
                ("eps", C.c_double), ("alpha", C.c_double), ("tau", C.c_double), ("nlevels", C.c_int),
                ("level", LevelInfo * MAX_LEVELS), ("p2p_pairs", C.c_int64), ("p2p_sym_pairs", C.c_int64),
                ("s2m_evals", C.c_int64),
                ("rank", C.c_int), ("nranks", C.c_int), ("owned_points", C.c_int64),
                ("source_level", C.c_int), ("launches", C.c_int), ("p2p_tile", C.c_int), ("next4_passes", C.c_int),
                ("p2p_rowskip", C.c_int), ("p2p_dead_frac", C.c_double), ("p2p_mixed_items", C.c_int64)]


class HFMMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libhfmm error {code}: {msg}")
        self.code = code


_lib = None


def load() -> C.CDLL:
    """Load libhfmm.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                          "(python -m paper_0911_4114_b200.build); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    vp, i64, dbl, ci = C.c_void_p, C.c_int64, C.c_double, C.c_int
    sig = {
        "hfmm_create": (ci, [C.POINTER(vp), ci]),
        "hfmm_set_dist": (ci, [vp, ci, ci, C.c_char_p]),
        "hfmm_nccl_unique_id": (ci, [vp]),
        "hfmm_build_tree": (ci, [vp, i64, vp, ci, vp, dbl]),
        "hfmm_precompute": (ci, [vp, dbl, dbl, dbl, dbl, C.c_uint]),
        "hfmm_matvec": (ci, [vp, vp, vp, ci, vp]),
        "hfmm_direct": (ci, [vp, vp, vp, ci, vp]),
        "hfmm_get_info": (ci, [vp, C.POINTER(Info)]),
        "hfmm_stage_times": (ci, [vp, vp]),
        "hfmm_debug_copy": (ci, [vp, ci, ci, vp, i64, C.POINTER(i64)]),
        "hfmm_last_error": (C.c_char_p, [vp]),
        "hfmm_destroy": (None, [vp]),
        "hfmm_level_quadrature": (ci, [dbl, dbl, dbl, dbl, C.POINTER(ci), C.POINTER(ci), C.POINTER(ci), vp, ci]),
        "hfmm_resample_workspace": (i64, [ci, ci, ci, ci, ci]),
        "hfmm_resample": (ci, [ci, ci, ci, ci, ci, vp, vp, vp, vp]),
        "hfmm_m2m_op": (ci, [ci, ci, ci, ci, ci, vp, vp, vp, vp, vp]),
        "hfmm_l2l_op": (ci, [ci, ci, ci, ci, ci, vp, vp, vp, vp, vp, vp]),
        "hfmm_m2l_op": (ci, [ci, i64, vp, vp, vp, vp, vp, vp, vp]),
        "hfmm_partition": (ci, [i64, vp, ci, vp, dbl, ci, i64, ci, vp, vp, vp]),
        "hfmm_halo_lists": (ci, [i64, vp, ci, vp, dbl, ci, i64, ci, ci, ci, vp, vp, vp, vp]),
        "hfmm_rep_grid": (ci, [dbl, dbl, dbl, C.POINTER(ci), C.POINTER(ci)]),
        "hfmm_m2l_op_plan": (ci, [ci, i64, vp, vp, vp, C.POINTER(vp)]),
        "hfmm_m2l_op_apply": (ci, [vp, vp, vp, vp, vp]),
        "hfmm_m2l_op_free": (None, [vp]),
        "hfmm_m2l_op_kind": (ci, [vp]),
        "hfmm_ragged_rows": (ci, [dbl, dbl, dbl, dbl, ci, ci, ci, vp]),
        "hfmm_vgroup_create": (ci, [C.POINTER(vp), ci]),
        "hfmm_set_dist_virtual": (ci, [vp, vp, ci]),
        "hfmm_vgroup_matvec": (ci, [vp, vp, vp, vp]),
        "hfmm_vgroup_destroy": (None, [vp]),
        "hfmm_set_next4": (ci, [ci]),
        "hfmm_set_fused": (ci, [ci]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    rc = load().hfmm_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc < 0:
        raise HFMMError(rc, "hfmm_nccl_unique_id")
    return buf.raw


def level_quadrature(kappa: float, a: float, eps_level: float, alpha: float = 0.8):
    """Host-only per-level quadrature (ell, N_theta, N_phi, ragged rows) -- no GPU needed."""
    lib = load()
    ell, nth, nph = C.c_int(), C.c_int(), C.c_int()
    cap = 4096
    rag = (C.c_int * cap)()
    rc = lib.hfmm_level_quadrature(kappa, a, eps_level, alpha, C.byref(ell), C.byref(nth), C.byref(nph),
                                   C.cast(rag, C.c_void_p), cap)
    if rc < 0:
        raise HFMMError(rc, "hfmm_level_quadrature failed")
    return ell.value, nth.value, nph.value, list(rag[: nth.value // 2 + 1])


def set_next4(on: bool) -> bool:
    """NEXT 4 coefficient-domain symmetric resampling on / off (process-wide; include/hfmm.h
    hfmm_set_next4).  Returns the previous setting."""
    return bool(load().hfmm_set_next4(1 if on else 0))


def set_fused(on: bool) -> bool:
    """Fused two-pass upward resampler on / off (process-wide; include/hfmm.h hfmm_set_fused)."""
    return bool(load().hfmm_set_fused(1 if on else 0))


def rep_grid(kappa: float, a: float, eps: float):
    """Host-only: (N_theta, N_phi) of a translation-only level (include/hfmm.h hfmm_rep_grid)."""
    nth, nph = C.c_int(), C.c_int()
    rc = load().hfmm_rep_grid(kappa, a, eps, C.byref(nth), C.byref(nph))
    if rc < 0:
        raise HFMMError(rc, "hfmm_rep_grid")
    return nth.value, nph.value


def ragged_rows(kappa: float, a: float, eps_level: float, alpha: float, ell: int, n_theta: int, n_phi_cap: int):
    """Host-only: per-row N_phi(theta_n) of an active level (include/hfmm.h hfmm_ragged_rows)."""
    out = np.zeros(n_theta, dtype=np.int32)
    rc = load().hfmm_ragged_rows(kappa, a, eps_level, alpha, ell, n_theta, n_phi_cap, out.ctypes.data)
    if rc < 0:
        raise HFMMError(rc, "hfmm_ragged_rows")
    return [int(v) for v in out]


def partition(xyz, depth, lo, size, L_f, K, nranks):
    """Host-only multi-GPU ownership rule: (level-2 cuts, sorted-point ranges, perm)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    n = xyz.shape[0]
    cuts = np.zeros(nranks + 1, dtype=np.int64)
    rng = np.zeros(2 * nranks, dtype=np.int64)
    perm = np.zeros(n, dtype=np.int64)
    rc = load().hfmm_partition(n, xyz.ctypes.data, depth, lo.ctypes.data, size, L_f, K, nranks,
                               cuts.ctypes.data, rng.ctypes.data, perm.ctypes.data)
    if rc < 0:
        raise HFMMError(rc, "hfmm_partition")
    return cuts, rng.reshape(nranks, 2), perm


def halo_lists(xyz, depth, lo, size, L_f, K, nranks, rank, level):
    """Host-only M2L halo lists of `rank` at `level` (the ones hfmm_precompute exchanges):
    (recv, send), each a list over peers q of sorted level-`level` box indices (Morton order)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    n = xyz.shape[0]
    ro = np.zeros(nranks + 1, dtype=np.int64)
    so = np.zeros(nranks + 1, dtype=np.int64)
    lib = load()
    args = (n, xyz.ctypes.data, depth, lo.ctypes.data, size, L_f, K, nranks, rank, level)
    rc = lib.hfmm_halo_lists(*args, ro.ctypes.data, so.ctypes.data, None, None)
    if rc < 0:
        raise HFMMError(rc, "hfmm_halo_lists")
    rb = np.zeros(max(int(ro[-1]), 1), dtype=np.int64)
    sb = np.zeros(max(int(so[-1]), 1), dtype=np.int64)
    rc = lib.hfmm_halo_lists(*args, ro.ctypes.data, so.ctypes.data, rb.ctypes.data, sb.ctypes.data)
    if rc < 0:
        raise HFMMError(rc, "hfmm_halo_lists")
    return ([rb[ro[q]:ro[q + 1]] for q in range(nranks)], [sb[so[q]:so[q + 1]] for q in range(nranks)])


def _ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


class HFMM:
    """One FMM plan on one GPU (see include/hfmm.h for the contract)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        rc = self.lib.hfmm_create(C.byref(h), device)
        if rc != 0:
            raise HFMMError(rc, self.lib.hfmm_last_error(None).decode())
        self.h = h
        self.device = int(device)
        self.n = 0
        self.last_rc = 0

    def _check(self, rc):
        self.last_rc = rc
        if rc < 0:
            raise HFMMError(rc, self.lib.hfmm_last_error(self.h).decode())
        return rc

    def close(self):
        if getattr(self, "h", None):
            self.lib.hfmm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_dist(self, rank: int, nranks: int, uid: Optional[bytes]):
        return self._check(self.lib.hfmm_set_dist(self.h, rank, nranks, uid))

    def build_tree(self, xyz: np.ndarray, depth: int, lo, size: float):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        self.n = xyz.shape[0]
        return self._check(self.lib.hfmm_build_tree(self.h, self.n, xyz.ctypes.data, depth, lo.ctypes.data, size))

    def precompute(self, kappa: float, eps: float, alpha: float = 0.8, tau: float = 0.0, flags: int = 0):
        return self._check(self.lib.hfmm_precompute(self.h, kappa, eps, alpha, tau, flags))

    def _check_vec(self, t, name: str, cuda: bool):
        """The library reads / writes exactly n complex128 values at the pointer: reject anything else
        (wrong dtype, strided view, wrong length, other device) before the call."""
        if hasattr(t, "data_ptr"):
            import torch
            ok = (t.dtype == torch.complex128 and t.is_contiguous() and tuple(t.shape) == (self.n,)
                  and bool(t.is_cuda) == cuda and (not cuda or t.device.index == self.device))
            what = f"{name}: dtype {t.dtype}, shape {tuple(t.shape)}, device {t.device}"
        else:
            ok = (isinstance(t, np.ndarray) and t.dtype == np.complex128 and t.flags.c_contiguous
                  and t.shape == (self.n,) and not cuda)
            what = f"{name}: {type(t).__name__} dtype {getattr(t, 'dtype', None)}, shape {getattr(t, 'shape', None)}"
        if not ok:
            where = f"cuda:{self.device}" if cuda else "host"
            raise HFMMError(-1, f"{what}; need a contiguous complex128 vector of shape ({self.n},) on {where}")

    def _apply(self, fn, q, out=None, stream=None, local=False, serial=False):
        mem_local = (HFMM_Y_LOCAL if local else 0) | (HFMM_SERIAL if serial else 0)
        if self.n <= 0:
            raise HFMMError(-5, "matvec before build_tree")
        if hasattr(q, "is_cuda") and q.is_cuda:
            import torch
            if out is None:
                out = torch.empty_like(q)
            self._check_vec(q, "q", True)
            self._check_vec(out, "out", True)
            s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
            if not s:
                s = 1  # torch's default stream is the legacy default stream (cudaStreamLegacy)
            self._check(fn(self.h, q.data_ptr(), out.data_ptr(), HFMM_DEVICE | mem_local, C.c_void_p(s)))
            return out
        if hasattr(q, "data_ptr"):  # CPU torch tensor (pinned or pageable): host path
            import torch
            if out is None:
                out = torch.empty_like(q)
            self._check_vec(q, "q", False)
            self._check_vec(out, "out", False)
            s = None if stream is None else C.c_void_p(stream or 1)  # 0 -> cudaStreamLegacy
            self._check(fn(self.h, q.data_ptr(), out.data_ptr(), HFMM_HOST | mem_local, s))
            return out
        q = np.ascontiguousarray(q, dtype=np.complex128)
        if out is None:
            out = np.empty_like(q)
        self._check_vec(q, "q", False)
        self._check_vec(out, "out", False)
        self._check(fn(self.h, q.ctypes.data, out.ctypes.data, HFMM_HOST | mem_local, None))
        return out

    def matvec(self, q, out=None, stream=None, local=False, serial=False):
        """y = A q (eqn:HelmholtzMatrixVector); numpy/CPU tensors use the host path."""
        return self._apply(self.lib.hfmm_matvec, q, out, stream, local, serial)

    def direct(self, q, out=None, stream=None):
        return self._apply(self.lib.hfmm_direct, q, out, stream)

    def info(self) -> dict:
        inf = Info()
        self._check(self.lib.hfmm_get_info(self.h, C.byref(inf)))
        levels = []
        for i in range(inf.nlevels):
            lv = inf.level[i]
            levels.append(dict(level=lv.level, a=lv.a, ell=lv.ell, n_theta=lv.n_theta, n_phi=lv.n_phi,
                               alpha=lv.alpha, K=lv.K,
                               F=lv.F, active=bool(lv.active), boxes=lv.boxes, m2l_pairs=lv.m2l_pairs,
                               rep=bool(lv.rep), ragged=bool(lv.ragged), m2l_block=bool(lv.m2l_block),
                               halo=bool(lv.halo), m_recv_boxes=int(lv.m_recv_boxes),
                               m_send_boxes=int(lv.m_send_boxes)))
        return dict(n=inf.n, depth=inf.depth, L_f=(None if inf.L_f < 0 else inf.L_f), kappa=inf.kappa,
                    eps=inf.eps, alpha=inf.alpha, tau=inf.tau, levels=levels, p2p_pairs=inf.p2p_pairs,
                    p2p_sym_pairs=inf.p2p_sym_pairs,
                    s2m_evals=inf.s2m_evals, rank=inf.rank, nranks=inf.nranks, owned_points=inf.owned_points,
                    source_level=(None if inf.source_level < 0 else inf.source_level), launches=inf.launches,
                    p2p_tile=inf.p2p_tile, next4_passes=inf.next4_passes,
                    p2p_rowskip=bool(inf.p2p_rowskip), p2p_dead_frac=inf.p2p_dead_frac,
                    p2p_mixed_items=int(inf.p2p_mixed_items))

    def stage_times(self):
        out = (C.c_double * 8)()
        self._check(self.lib.hfmm_stage_times(self.h, C.cast(out, C.c_void_p)))
        keys = ["s2m", "m2m", "m2l", "l2l", "l2t", "p2p", "total"]
        return {k: out[i] for i, k in enumerate(keys)}

    def debug(self, what: int, level: int = 0) -> np.ndarray:
        need = C.c_int64()
        self._check(self.lib.hfmm_debug_copy(self.h, what, level, None, 0, C.byref(need)))
        if what in (6, 7):
            buf = np.empty(need.value // 8, dtype=np.int64)
        else:
            buf = np.empty(need.value // 16, dtype=np.complex128)
        if need.value:
            self._check(self.lib.hfmm_debug_copy(self.h, what, level, buf.ctypes.data, need.value, C.byref(need)))
        if what == 7:
            buf = buf.reshape(-1, 4)
        return buf


class VirtualGroup:
    """nranks plans on one device acting as the ranks of a multi-GPU run (test mode; include/hfmm.h
    hfmm_vgroup_*).  Bind plans with `bind(plan, rank)` before their build_tree."""

    def __init__(self, nranks: int):
        self.lib = load()
        h = C.c_void_p()
        rc = self.lib.hfmm_vgroup_create(C.byref(h), nranks)
        if rc != 0:
            raise HFMMError(rc, "hfmm_vgroup_create")
        self.h, self.nranks, self.plans = h, nranks, [None] * nranks

    def bind(self, plan: "HFMM", rank: int):
        plan._check(self.lib.hfmm_set_dist_virtual(plan.h, self.h, rank))
        self.plans[rank] = plan

    def matvec(self, q, out=None, stream=None):
        """q: device complex128 [n] -> [nranks][n] (every rank's output vector)."""
        import torch
        n = self.plans[0].n
        self.plans[0]._check_vec(q, "q", True)
        if out is None:
            out = torch.empty((self.nranks, n), dtype=torch.complex128, device=q.device)
        if out.dtype != torch.complex128 or not out.is_contiguous() or tuple(out.shape) != (self.nranks, n):
            raise HFMMError(-1, f"out must be a contiguous complex128 tensor of shape ({self.nranks}, {n})")
        rc = self.lib.hfmm_vgroup_matvec(self.h, q.data_ptr(), out.data_ptr(), _stream(stream))
        if rc < 0:
            raise HFMMError(rc, "hfmm_vgroup_matvec: " + self.plans[0].lib.hfmm_last_error(self.plans[0].h).decode())
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.hfmm_vgroup_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    return C.c_void_p(stream or 1)  # 0 (torch default stream) -> cudaStreamLegacy


def resample(inp, nth, nph, nth2, nph2, out, work=None, stream=None):
    """Batched 5-step resample of device fields [B][nth][nph/2] -> [B][nth2][nph2/2] (torch tensors)."""
    lib = load()
    rc = lib.hfmm_resample(inp.shape[0], nth, nph, nth2, nph2, inp.data_ptr(), out.data_ptr(),
                           None if work is None else work.data_ptr(), _stream(stream))
    if rc < 0:
        raise HFMMError(rc, "hfmm_resample")
    return out


def resample_workspace(nbatch, nth, nph, nth2, nph2) -> int:
    return load().hfmm_resample_workspace(nbatch, nth, nph, nth2, nph2)


def m2m_op(child, shift, parent, nth, nph, nth2, nph2, work=None, stream=None):
    lib = load()
    rc = lib.hfmm_m2m_op(parent.shape[0], nth, nph, nth2, nph2, child.data_ptr(), shift.data_ptr(),
                         parent.data_ptr(), None if work is None else work.data_ptr(), _stream(stream))
    if rc < 0:
        raise HFMMError(rc, "hfmm_m2m_op")
    return parent


def l2l_op(parent, shift, incoming, child_out, nth, nph, nth2, nph2, work=None, stream=None):
    lib = load()
    rc = lib.hfmm_l2l_op(parent.shape[0], nth, nph, nth2, nph2, parent.data_ptr(), shift.data_ptr(),
                         None if incoming is None else incoming.data_ptr(), child_out.data_ptr(),
                         None if work is None else work.data_ptr(), _stream(stream))
    if rc < 0:
        raise HFMMError(rc, "hfmm_l2l_op")
    return child_out


def m2l_op(row, src, oid, T, M, out, stream=None):
    lib = load()
    nbox = row.shape[0] - 1
    K = M.shape[-1] if M.dim() == 2 else M.shape[1] * M.shape[2]
    rc = lib.hfmm_m2l_op(nbox, K, row.data_ptr(), src.data_ptr(), oid.data_ptr(), T.data_ptr(), M.data_ptr(),
                         out.data_ptr(), _stream(stream))
    if rc < 0:
        raise HFMMError(rc, "hfmm_m2l_op")
    return out


class M2LOp:
    """Sibling-group M2L plan built once from a HOST CSR (numpy int32 row / src / oid), applied to
    device tensors (T [316][K], M and out [nbox][K], complex128) -- include/hfmm.h hfmm_m2l_op_plan."""

    def __init__(self, row, src, oid, K: int):
        self.lib = load()
        row, src, oid = (np.ascontiguousarray(a, dtype=np.int32) for a in (row, src, oid))
        h = C.c_void_p()
        rc = self.lib.hfmm_m2l_op_plan(len(row) - 1, K, _ptr(row), _ptr(src), _ptr(oid), C.byref(h))
        if rc < 0:
            raise HFMMError(rc, "hfmm_m2l_op_plan")
        self.h = h

    @property
    def kind(self) -> str:
        """"block" (parent-block kernel) or "list" (merged-list kernel): hfmm_m2l_op_kind."""
        return {1: "block", 0: "list"}[self.lib.hfmm_m2l_op_kind(self.h)]

    def apply(self, T, M, out, stream=None):
        rc = self.lib.hfmm_m2l_op_apply(self.h, T.data_ptr(), M.data_ptr(), out.data_ptr(), _stream(stream))
        if rc < 0:
            raise HFMMError(rc, "hfmm_m2l_op_apply")
        return out

    def close(self):
        if getattr(self, "h", None):
            self.lib.hfmm_m2l_op_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
