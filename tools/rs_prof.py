"""Two C2 resamples (65,536 boxes) for ncu: python tools/rs_prof.py B [down]"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0911_4114_b200 as hf
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
down = len(sys.argv) > 2 and sys.argv[2] == "down"
n = 65536
a, b = (2 * B, 2 * B), (4 * B, 4 * B)
if down:
    a, b = b, a
x = torch.randn(n, a[0] * a[1] // 2, dtype=torch.complex128, device="cuda")
y = torch.zeros(n, b[0] * b[1] // 2, dtype=torch.complex128, device="cuda")
for _ in range(2):
    hf.resample(x, a[0], a[1], b[0], b[1], y)
torch.cuda.synchronize()
