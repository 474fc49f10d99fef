#!/bin/bash
# NEXT 4 A/B (same box): C2 operators B8/B16/B32 and the C4 / C3 matvecs with the coefficient-domain
# symmetric kernels (HFMM_NEXT4=1) vs the default single-pass / two-pass 5-step kernels.
mkdir -p gpurun_out
out=gpurun_out/next4_ab.txt
: > $out
for rep in 1 2; do
  for v in 0 1; do
    HFMM_NEXT4=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops 8,16,32 --extra C3 > gpurun_out/n4ab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/n4ab_{v}.log").read().strip().splitlines()[-1])
ops = d["operators"]
row = [f"NEXT4={v}", f"C4 {d['ms_per_step']:.2f} ms", f"C3 {d['other_configs']['C3']['ms_per_matvec']:.3f} ms"]
for B in ("B8", "B16", "B32"):
    o = ops[B]
    row.append(f"{B} interp {o['interp']['ms']:.3f} anterp {o['anterp']['ms']:.3f} m2m {o['m2m']['ms']:.3f} l2l {o['l2l']['ms']:.3f}")
print(" | ".join(row))
PY
  done
done
cat $out
