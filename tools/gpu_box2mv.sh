mkdir -p gpurun_out
: > gpurun_out/box2mv.log
echo "[gpu tests] $(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> gpurun_out/box2mv.log
for rep in 1 2; do
  for v in "" prev; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/box2mv_$v.log 2>&1
    python - "$v" >> gpurun_out/box2mv.log <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/box2mv_{sys.argv[1]}.log").read().strip().splitlines()[-1])
oc = d.get("other_configs", {})
print(sys.argv[1] or "default", "C4", round(d["ms_per_step"], 2), d["gpu_launches"], "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1))
PY
  done
done
cat gpurun_out/box2mv.log
