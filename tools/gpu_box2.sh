# single-pass small-grid upward resample: parity (C2 + matvec) and A/B vs the previous commit
mkdir -p gpurun_out
: > gpurun_out/box2.log
echo "[c2] $(timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/box2.log
echo "[parity] $(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1)" >> gpurun_out/box2.log
for rep in 1 2; do
  for v in "" prev; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 8 16 >> gpurun_out/box2.log 2>&1
    HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/box2_bench_$v.log 2>&1
    python - "$v" >> gpurun_out/box2.log <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/box2_bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("C4", sys.argv[1] or "default", round(d["ms_per_step"], 2), d["gpu_launches"])
PY
  done
done
cat gpurun_out/box2.log
