"""A/B of the sibling-group M2L on the C2 lattice (65,536 boxes x 189 partners): ms and FP64 fraction."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0911_4114_b200 as hf
from workloads import c2_lattice, c2_grids
_, row, src, oid, _ = c2_lattice()
for B in (16, 32, 64):
    (nth, nph), _ = c2_grids(B)
    K = nth * nph // 2
    M = torch.randn(65536, K, dtype=torch.complex128, device="cuda")
    T = torch.randn(316, K, dtype=torch.complex128, device="cuda")
    I = torch.empty_like(M)
    op = hf.M2LOp(row, src, oid, K)
    op.apply(T, M, I)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        torch.cuda.synchronize(); e0.record(); op.apply(T, M, I); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    print(f"{os.path.basename(os.environ.get('HFMM_LIB', 'default'))} [{op.kind}] B{B}: {t:.3f} ms  "
          f"{8 * 189 * 65536 * K / t / 1e9 / 37.22:.3f} of FP64", flush=True)
    del M, T, I; op.close(); torch.cuda.empty_cache()
