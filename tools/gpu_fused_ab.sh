#!/bin/bash
# Fused two-pass upward resampler A/B (same box): C2 operators, fused (default build, 3 CTAs/SM),
# fused with 2 CTAs/SM (libhfmm_fmb2.so), and HFMM_FUSED=0 (two-pass kernels).
mkdir -p gpurun_out
out=gpurun_out/fused_ab.txt
: > $out
for rep in 1 2; do
  for v in f1 f0 fmb2; do
    lib=""; fu=1
    [ "$v" = fmb2 ] && lib="$PWD/paper_0911_4114_b200/libhfmm_fmb2.so"
    [ "$v" = f0 ] && fu=0
    HFMM_LIB=$lib HFMM_FUSED=$fu timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --ops 32,64 --extra "" > gpurun_out/fuab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/fuab_{v}.log").read().strip().splitlines()[-1])
ops = d["operators"]
print(v, "C4", round(d["ms_per_step"], 2), " | ".join(f"{B}: interp {ops[B]['interp']['ms']:.3f} ms ({ops[B]['interp']['frac_hbm']:.3f} HBM) m2m {ops[B]['m2m']['ms']:.3f} ms" for B in ("B32", "B64")))
PY
  done
done
cat $out
