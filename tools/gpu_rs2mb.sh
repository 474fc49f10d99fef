# register-resident resample passes: 3 vs 4 resident CTAs per SM (launch bounds), C2 operators
mkdir -p gpurun_out
L=$PWD/paper_0911_4114_b200
: > gpurun_out/rs2mb.log
for r in 1 2; do
for v in "" rs2mb4; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 32 64 >> gpurun_out/rs2mb.log 2>&1
done; done
HFMM_LIB=$L/libhfmm_rs2mb4.so timeout 900 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -2 >> gpurun_out/rs2mb.log
cat gpurun_out/rs2mb.log
