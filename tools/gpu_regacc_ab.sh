mkdir -p gpurun_out
L=$PWD/paper_0911_4114_b200
for v in regacc regacc2; do
HFMM_LIB=$L/libhfmm_$v.so timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_baseline_parity.py -x -q -k "c2 or grid_pairs or operator" > gpurun_out/regacc_pytest_$v.log 2>&1; tail -1 gpurun_out/regacc_pytest_$v.log
done
: > gpurun_out/regacc_ab.log
for r in 1 2; do
for v in "" regacc regacc2; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 32 64 >> gpurun_out/regacc_ab.log 2>&1
done; done
cat gpurun_out/regacc_ab.log
