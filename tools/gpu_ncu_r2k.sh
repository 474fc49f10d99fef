# session-4 full captures: the dominant kernel (P2P symmetric, C4 timed step) and the new L2T v3
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r2k_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_sym_kernel -s 6 -c 1 \
  -o gpurun_out/r2k_p2p python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r2k_ncu_p2p.log 2>&1
ncu -i gpurun_out/r2k_p2p.ncu-rep --page details --csv > gpurun_out/r2k_p2p_details.csv 2>/dev/null
ncu -i gpurun_out/r2k_p2p.ncu-rep --page raw --csv > gpurun_out/r2k_p2p_raw.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:l2t_warp3 -s 2 -c 1 \
  -o gpurun_out/r2k_l2t python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r2k_ncu_l2t.log 2>&1
ncu -i gpurun_out/r2k_l2t.ncu-rep --page details --csv > gpurun_out/r2k_l2t_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/r2k_*
