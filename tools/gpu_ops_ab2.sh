# C2 operator A/B with a parity check per variant: VARIANTS="a b" bash tools/gpu_ops_ab2.sh
mkdir -p gpurun_out
: > gpurun_out/ops_ab.log
for v in "" $VARIANTS; do
  lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
  echo "[$v] $(HFMM_LIB=$lib timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/ops_ab.log
done
for rep in 1 2; do
  for v in "" $VARIANTS; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 8 16 32 64 >> gpurun_out/ops_ab.log 2>&1
  done
done
cat gpurun_out/ops_ab.log
