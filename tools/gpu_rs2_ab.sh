# register-resident resample passes (HFMM_RS2=1) vs tiled: parity + C2 operator timings, same box
mkdir -p gpurun_out
: > gpurun_out/rs2_ab.log
echo "[rs2] $(HFMM_RS2=1 timeout 600 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -1)" >> gpurun_out/rs2_ab.log
echo "[rs2 parity] $(HFMM_RS2=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1)" >> gpurun_out/rs2_ab.log
for rep in 1 2; do
  for v in 0 1; do
    echo "RS2=$v" >> gpurun_out/rs2_ab.log
    HFMM_RS2=$v timeout 600 python tools/ops_ab.py 8 16 32 64 >> gpurun_out/rs2_ab.log 2>&1
  done
done
cat gpurun_out/rs2_ab.log
