# A/B timing of kernel variants (HFMM_LIB) on the C4 bench; parity of each variant first
mkdir -p gpurun_out
for v in "" noprio; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or deep or c1" 2>&1 | tail -2 > gpurun_out/ab_test_$v.log
  HFMM_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/ab_bench_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
t = open(f"gpurun_out/ab_test_{v}.log").read().strip().splitlines()[-1]
try:
    d = json.loads(open(f"gpurun_out/ab_bench_{v}.log").read().strip().splitlines()[-1])
    print(f"variant[{v}] tests: {t} | ms {d['ms_per_step']:.2f} p2p {d['stages_ms']['p2p']:.2f} frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(f"variant[{v}] tests: {t} | ERR {e}")
PY
done
