# L2-sized batching of the two-pass resample (operator entry points): HFMM_RS_L2_MB A/B, same box
mkdir -p gpurun_out
: > gpurun_out/l2b.log
echo "[c2] $(timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/l2b.log
for rep in 1 2; do
  for mb in 0 16 24 48; do
    echo "L2_MB=$mb" >> gpurun_out/l2b.log
    HFMM_RS_L2_MB=$mb timeout 600 python tools/ops_ab.py 8 16 32 64 >> gpurun_out/l2b.log 2>&1
  done
done
cat gpurun_out/l2b.log
