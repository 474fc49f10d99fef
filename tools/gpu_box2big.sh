mkdir -p gpurun_out
: > gpurun_out/box2big.log
echo "[c2 big] $(HFMM_BOX2_BIG=1 timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/box2big.log
for rep in 1 2; do
  for v in 0 1; do
    echo "BIG=$v" >> gpurun_out/box2big.log
    HFMM_BOX2_BIG=$v timeout 600 python tools/ops_ab.py 32 >> gpurun_out/box2big.log 2>&1
  done
done
cat gpurun_out/box2big.log
