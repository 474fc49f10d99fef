#!/usr/bin/env python3
"""List every FP64 loop (backward branch) of the kernels matching a name, innermost first, with the
FP64 slot cost of tools/sass_fp64_cost.py:  sass_loops.py <object> <function-substring>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_fp64_cost as S  # noqa: E402

path, fsub = sys.argv[1], sys.argv[2]
for name, body in S.functions(path).items():
    if fsub not in name:
        continue
    loops = []
    for i, (addr, op, ops) in enumerate(body):
        if op.startswith("BRA") and ops:
            try:
                tgt = int(ops[-1].split()[-1], 16)
            except ValueError:
                continue
            if tgt < addr:
                lo = next(j for j, b in enumerate(body) if b[0] >= tgt)
                seg = body[lo:i + 1]
                n = sum(1 for b in seg if b[1].split(".")[0] in S.FP64)
                if n:
                    loops.append((len(seg), seg))
    print(name)
    for L, seg in sorted(loops, key=lambda x: x[0]):
        slots, nfp, n3, reads, mix = S.cost(seg)
        top = ", ".join(f"{k} {v}" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:8])
        print(f"  loop {L} insns, FP64 {nfp} ({n3} 3-reg), slots {slots:.1f}: {top}")
