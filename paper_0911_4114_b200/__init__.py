"""paper_0911_4114_b200 -- B200-native Fourier-basis Helmholtz FMM matvec (Cecka & Darve, arXiv 0911.4114).

The product is libhfmm.so (C ABI, include/hfmm.h) with hand-written sm_100a CUDA kernels;
this package holds its sources (csrc/), the in-tree build (build.py) and a thin ctypes
binding (binding.py).  Nothing here imports oracle/ (test infrastructure only).
"""
from .binding import (HFMM, HFMMError, HFMM_ALPHA_FIXED, HFMM_EPS_ABSOLUTE, HFMM_FORCE_ALL_LEVELS,
                      HFMM_RAGGED, HFMM_DETERMINISTIC, HFMM_ATOMIC_NEAR, HFMM_SOURCE_AT_DEPTH, HFMM_SOURCE_AT_LF, HFMM_W_BREAKDOWN, HFMM_W_NO_FARFIELD, EXPORTED,
                      LIB_PATH, M2LOp, halo_lists, l2l_op, level_quadrature, load, m2l_op, m2m_op, nccl_unique_id, partition,
                      ragged_rows, rep_grid, resample, resample_workspace, VirtualGroup, set_next4, set_fused)

__all__ = ["HFMM", "HFMMError", "HFMM_ALPHA_FIXED", "HFMM_EPS_ABSOLUTE", "HFMM_FORCE_ALL_LEVELS",
           "HFMM_SOURCE_AT_DEPTH", "HFMM_SOURCE_AT_LF", "HFMM_RAGGED", "HFMM_DETERMINISTIC", "HFMM_ATOMIC_NEAR", "ragged_rows", "rep_grid", "M2LOp", "HFMM_W_BREAKDOWN", "HFMM_W_NO_FARFIELD", "EXPORTED", "LIB_PATH", "l2l_op", "level_quadrature",
           "halo_lists", "load", "m2l_op", "m2m_op", "nccl_unique_id", "partition", "resample", "resample_workspace", "VirtualGroup", "set_next4", "set_fused"]
