# C2 operator A/B of library variants, alternating to expose box noise: VARIANTS="a b" bash tools/gpu_ops_ab.sh
mkdir -p gpurun_out
: > gpurun_out/ops_ab.log
for rep in 1 2; do
  for v in "" $VARIANTS; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 8 16 64 >> gpurun_out/ops_ab.log 2>&1
  done
done
cat gpurun_out/ops_ab.log
