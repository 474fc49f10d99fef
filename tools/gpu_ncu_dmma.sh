mkdir -p gpurun_out
timeout 300 python tools/m2l_one.py 32 || exit 1
timeout 600 ncu --set full --clock-control none -k regex:m2l_dmma -c 1 -o gpurun_out/ncu_dmma python tools/m2l_one.py 32 > gpurun_out/ncu_dmma.log 2>&1
ncu -i gpurun_out/ncu_dmma.ncu-rep --page details --csv > gpurun_out/ncu_dmma_details.csv 2>/dev/null
ncu -i gpurun_out/ncu_dmma.ncu-rep --page raw --csv > gpurun_out/ncu_dmma_raw.csv 2>/dev/null
ls -la gpurun_out/ncu_dmma*
