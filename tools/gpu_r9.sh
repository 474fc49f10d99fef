# parent-block M2L (parity + A/B vs merged-list), full-N direct test, TAB=2048 P2P A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q -k "m2l" 2>&1 | tail -5 > gpurun_out/r9_pytest_m2l.log
timeout 600 python tools/m2l_ab.py > gpurun_out/r9_m2l_ab.log 2>&1
HFMM_M2L_LIST=1 timeout 600 python tools/m2l_ab.py >> gpurun_out/r9_m2l_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "every_output" 2>&1 | tail -5 > gpurun_out/r9_pytest_full.log
for v in "" tab2k; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small or deep or c1" 2>&1 | tail -2 > gpurun_out/ab_test_$v.log
  HFMM_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ab_bench_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
t = open(f"gpurun_out/ab_test_{v}.log").read().strip().splitlines()[-1]
try:
    d = json.loads(open(f"gpurun_out/ab_bench_{v}.log").read().strip().splitlines()[-1])
    print(f"variant[{v}] tests: {t} | ms {d['ms_per_step']:.2f} p2p {d['stages_ms']['p2p']:.2f} frac {d['roofline']['frac']:.3f} serial {d['roofline'].get('frac_serial')}")
except Exception as e:
    print(f"variant[{v}] tests: {t} | ERR {e}")
PY
done
cat gpurun_out/r9_pytest_m2l.log gpurun_out/r9_m2l_ab.log gpurun_out/r9_pytest_full.log
