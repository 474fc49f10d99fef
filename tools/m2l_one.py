"""One C2 M2L operator call at bandwidth B (default 32) -- for ncu captures of the M2L kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0911_4114_b200 as hf
from workloads import c2_lattice, c2_grids
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
_, row, src, oid, _ = c2_lattice()
(nth, nph), _ = c2_grids(B)
K = nth * nph // 2
M = torch.randn(65536, K, dtype=torch.complex128, device="cuda")
T = torch.randn(316, K, dtype=torch.complex128, device="cuda")
I = torch.empty_like(M)
op = hf.M2LOp(row, src, oid, K)
for _ in range(2):
    op.apply(T, M, I)
torch.cuda.synchronize()
print(op.kind, "ok")
