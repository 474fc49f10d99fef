"""A/B of the resample operators (C2 sizes, 65,536 boxes): interp / anterp ms and HBM fraction."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_0911_4114_b200 as hf
tag = os.path.basename(os.environ.get("HFMM_LIB", "default"))
for B in (8, 16, 32, 64):
    a, b = (2 * B, 2 * B), (4 * B, 4 * B)
    K, K2 = a[0] * a[1] // 2, b[0] * b[1] // 2
    x = torch.randn(65536, K, dtype=torch.complex128, device="cuda")
    y = torch.empty(65536, K2, dtype=torch.complex128, device="cuda")
    w = torch.empty(max(hf.resample_workspace(65536, *a, *b), hf.resample_workspace(65536, *b, *a)), dtype=torch.uint8, device="cuda")
    res = []
    for (src, dst, g1, g2) in ((x, y, a, b), (y, x, b, a)):
        hf.resample(src, *g1, *g2, dst, work=w)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(3):
            torch.cuda.synchronize(); e0.record(); hf.resample(src, *g1, *g2, dst, work=w); e1.record(); torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t = statistics.median(ms)
        res.append(f"{t:.3f} ms ({65536 * (K + K2) * 16 / t / 1e6 / 6548.5:.3f})")
    print(f"{tag} B{B}: interp {res[0]}  anterp {res[1]}", flush=True)
    del x, y, w; torch.cuda.empty_cache()
