mkdir -p gpurun_out
: > gpurun_out/rs2_pf.log
echo "[c2] $(timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/rs2_pf.log
echo "[parity] $(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1)" >> gpurun_out/rs2_pf.log
for rep in 1 2; do
  for v in "" nopf; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 16 32 64 >> gpurun_out/rs2_pf.log 2>&1
  done
done
cat gpurun_out/rs2_pf.log
