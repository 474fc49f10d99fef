mkdir -p gpurun_out
L=$PWD/paper_0911_4114_b200
HFMM_LIB=$L/libhfmm_dmma.so timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q -k "m2l" > gpurun_out/dmma_pytest.log 2>&1; tail -2 gpurun_out/dmma_pytest.log
: > gpurun_out/dmma_ab.log
for r in 1 2; do
for v in dmma ""; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/m2l_ab.py >> gpurun_out/dmma_ab.log 2>&1
done; done
cat gpurun_out/dmma_ab.log
