"""CPU oracle for the Fourier-basis Helmholtz FMM matvec (Cecka & Darve, arXiv 0911.4114).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
(paper_0911_4114_b200/, libhfmm.so) never imports, links or executes it, and
shares no code, header, table or constant generator with it.

Plain, slow, obviously-correct numpy float64/complex128, each function citing
the PAPER.md passage it follows ("P:n" = line n of /root/reference/PAPER.md).
Fourier work uses explicit dense DFT matrices (no FFT), so it is independent of
the GPU's shared-memory FFTs.

Modules
  specfun   j_n, y_n, h_n, J_n, P_n
  plan      ell (EBF + Collino), Alg. 2, Alg. 3, rounding,
            F_l admissibility, L_f
  transfer  Alg. 1 bandlimited modified transfer function
  resample  1-D Fourier inter/anterpolation, 5-step 2-D
  tree      octree, neighbour and interaction lists
  fmm       S2M, M2M, M2L, L2L, L2T, P2P
  direct    compensated O(N^2) direct sum
  rig       single-pair error rig eps_T / eps_G / eps_I

Parity status: every function is pinned by a
-m "not gpu" test except the absolute FMM output on the BASELINE configs, which
has no printed value; it is pinned indirectly (vs direct summation within eps,
and stage identities).
"""
