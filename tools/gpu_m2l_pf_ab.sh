#!/bin/bash
# M2L parent-block kernel: 16-direction chunks, 2 groups per warp, cp.async prefetch of the next
# neighbour parent (default build) vs the 32-direction kernel (libhfmm_pf0.so), same box.
mkdir -p gpurun_out
out=gpurun_out/m2l_pf_ab.txt
: > $out
echo "[pf16 parity] $(timeout 900 python -m pytest tests/test_gpu_c2.py -k m2l -q 2>&1 | tail -1)" >> $out
echo "[pf16 parity] $(timeout 900 python -m pytest tests/test_gpu_parity.py -k 'm2l_kernels or small or cube' -q 2>&1 | tail -1)" >> $out
for rep in 1 2; do
  for v in "" pf0; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --ops 8,16,32,64 --extra C5 > gpurun_out/m2lpf_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/m2lpf_{v}.log").read().strip().splitlines()[-1])
ops = d["operators"]
print(v or "pf16", "C4", round(d["ms_per_step"], 2), "C5", round(d["other_configs"]["C5"]["ms_per_matvec"], 1), " ".join(f"{B}: m2l {ops[B]['m2l']['ms']:.3f} ms fp64 {ops[B]['m2l']['frac_fp64']:.3f}" for B in ("B8", "B16", "B32", "B64")))
PY
  done
done
cat $out
