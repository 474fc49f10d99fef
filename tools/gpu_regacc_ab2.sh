mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_baseline_parity.py -x -q -k "c2 or grid_pairs or operator" > gpurun_out/regacc2_pytest.log 2>&1; tail -1 gpurun_out/regacc2_pytest.log
: > gpurun_out/regacc_ab2.log
for r in 1 2 3; do HFMM_LIB= timeout 600 python tools/ops_ab.py 32 64 >> gpurun_out/regacc_ab2.log 2>&1; done
cat gpurun_out/regacc_ab2.log
