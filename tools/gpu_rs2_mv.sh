# RS2 on the matvec sizes: full parity + C3/C4/C5 timings with HFMM_RS2=0/1, and the C2 A/B
mkdir -p gpurun_out
: > gpurun_out/rs2_mv.log
echo "[rs2 gpu tests] $(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/rs2_mv.log
for v in 0 1 0 1; do
  HFMM_RS2=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/rs2_mv_$v.log 2>&1
  python - $v >> gpurun_out/rs2_mv.log <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/rs2_mv_{sys.argv[1]}.log").read().strip().splitlines()[-1])
oc = d.get("other_configs", {})
print("RS2=" + sys.argv[1], "C4", round(d["ms_per_step"], 2), "C3", round(oc.get("C3", {}).get("ms_per_matvec", 0), 3), "C5", round(oc.get("C5", {}).get("ms_per_matvec", 0), 1))
PY
done
cat gpurun_out/rs2_mv.log
bash tools/gpu_rs2_ab.sh | tail -18
