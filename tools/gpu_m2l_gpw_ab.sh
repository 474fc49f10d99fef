#!/bin/bash
# M2L parent-block kernel: 2 sibling groups per warp (default build) vs 1 (libhfmm_gpw1.so), same box.
# Parity first (C2 M2L vs oracle, matvec M2L kernels vs oracle), then the C2 operator bench.
mkdir -p gpurun_out
out=gpurun_out/m2l_gpw_ab.txt
: > $out
echo "[gpw2 parity] $(timeout 900 python -m pytest tests/test_gpu_c2.py -k m2l -q 2>&1 | tail -1)" >> $out
echo "[gpw2 parity] $(timeout 900 python -m pytest tests/test_gpu_parity.py -k m2l_kernels -q 2>&1 | tail -1)" >> $out
for rep in 1 2; do
  for v in "" gpw1; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --ops 8,16,32,64 --extra "" > gpurun_out/m2lab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/m2lab_{v}.log").read().strip().splitlines()[-1])
ops = d["operators"]
print(v or "gpw2", "C4", round(d["ms_per_step"], 2), " ".join(f"{B}: m2l {ops[B]['m2l']['ms']:.3f} ms fp64 {ops[B]['m2l']['frac_fp64']:.3f}" for B in ("B8", "B16", "B32", "B64")))
PY
  done
done
cat $out
