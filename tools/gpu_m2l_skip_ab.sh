# M2L parent-block: zero-table skip (+ split accumulators) A/B on C2, with parity of the skip build
mkdir -p gpurun_out
L=$PWD/paper_0911_4114_b200
HFMM_LIB=$L/libhfmm_skip.so timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q -k "m2l" 2>&1 | tail -3 > gpurun_out/m2lskip_pytest.log
: > gpurun_out/m2lskip.log
for r in 1 2; do
for v in "" skip skipsplit; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/m2l_ab.py >> gpurun_out/m2lskip.log 2>&1
done; done
cat gpurun_out/m2lskip_pytest.log gpurun_out/m2lskip.log
