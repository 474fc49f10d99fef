mkdir -p gpurun_out
: > gpurun_out/m2l_split.log
echo "[split12 c2] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_split12.so timeout 600 python -m pytest tests/test_gpu_c2.py -x -q -k m2l 2>&1 | tail -1)" >> gpurun_out/m2l_split.log
for rep in 1 2; do
  for v in "" split split12; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 600 python tools/m2l_ab.py >> gpurun_out/m2l_split.log 2>&1
  done
done
cat gpurun_out/m2l_split.log
