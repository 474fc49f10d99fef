# parent-block M2L variants: parity (default) + C2 timing of each variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q -k "m2l" 2>&1 | tail -3 > gpurun_out/m2lab_pytest.log
: > gpurun_out/m2lab.log
for v in "" dpf dpf12 w12; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/m2l_ab.py >> gpurun_out/m2lab.log 2>&1
done
cat gpurun_out/m2lab_pytest.log gpurun_out/m2lab.log
