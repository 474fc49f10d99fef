mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q -k "grid_pairs or c2 or operator or small or deep or c4_small" > gpurun_out/wide_pytest.log 2>&1; tail -1 gpurun_out/wide_pytest.log
L=$PWD/paper_0911_4114_b200
: > gpurun_out/wide_ab.log
for r in 1 2; do for v in "" narrow; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  echo "== ${v:-wide}" >> gpurun_out/wide_ab.log
  HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 8 16 >> gpurun_out/wide_ab.log 2>&1
  HFMM_LIB=$lib timeout 300 python tools/c5acc_stages.py C4 x serial | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4 serial', {k: round(v,3) for k,v in d['stages_ms'].items()})" >> gpurun_out/wide_ab.log 2>&1
  HFMM_LIB=$lib timeout 300 python tools/c5acc_stages.py C3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', {k: round(v,3) for k,v in d['stages_ms'].items()})" >> gpurun_out/wide_ab.log 2>&1
done; done
cat gpurun_out/wide_ab.log
