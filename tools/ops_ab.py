"""C2 operator timings of the library HFMM_LIB points at (A/B of kernel variants in one GPU call):
    HFMM_LIB=... python tools/ops_ab.py 8 16 64"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

Bs = [int(b) for b in sys.argv[1:]] or [8, 16, 64]
r = bench.bench_operators(Bs, reps=5)
tag = os.path.basename(os.environ.get("HFMM_LIB", "") or "default")
for B in Bs:
    d = r[f"B{B}"]
    print(tag, f"B{B}", " ".join(f"{k} {v['ms']:.3f}" for k, v in d.items()), flush=True)
