# ncu --set full of the C2 operator kernels themselves (not the C4 far chain): M2L parent-block
# (B16), interp rows/cols (B64, B16)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_dense -c 1 -o gpurun_out/m2l_dense_B16 python tools/m2l_ab.py > gpurun_out/ncu_m2l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_kernel" -c 2 -o gpurun_out/interp_B64 python tools/rs_prof.py 64 > gpurun_out/ncu_rs64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_kernel" -c 2 -o gpurun_out/interp_B16 python tools/rs_prof.py 16 > gpurun_out/ncu_rs16.log 2>&1
ls -la gpurun_out/*.ncu-rep
