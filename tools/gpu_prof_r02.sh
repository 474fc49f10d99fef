#!/bin/bash
# Round-2 profiles: bench (plain), then the ncu launch list of the same command (cold, serialised,
# clock-control none), then one full ncu capture of the dominant kernel (P2P symmetric) and of the
# C2 B64 M2L / interpolation passes.  Each profile command runs only after its plain command exited 0.
mkdir -p gpurun_out
set -o pipefail
python bench.py --steps 5 --warmup 3 --ops "" --extra "" > gpurun_out/r02_bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:p2p_sym_kernel -s 20 -c 1 \
  -o gpurun_out/r02_p2p_sym python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r02_ncu_p2p.log 2>&1
ncu -i gpurun_out/r02_p2p_sym.ncu-rep --page raw --csv > gpurun_out/r02_p2p_sym_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_p2p_sym.ncu-rep --page details --csv > gpurun_out/r02_p2p_sym_details.csv 2>/dev/null
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops 64 --extra "" > gpurun_out/r02_ops_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"m2l_dense|rows2_kernel|cols2_kernel" -s 6 -c 6 \
  -o gpurun_out/r02_ops_b64 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops 64 --extra "" > gpurun_out/r02_ncu_ops.log 2>&1
ncu -i gpurun_out/r02_ops_b64.ncu-rep --page raw --csv > gpurun_out/r02_ops_b64_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_ops_b64.ncu-rep --page details --csv > gpurun_out/r02_ops_b64_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | tail -20
