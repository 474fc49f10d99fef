# Full round check: GPU tests, bench (with operators + cpu baseline), launch list, ncu captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader; nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_sym -s 2 -c 1 -o gpurun_out/p2p_sym_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rows_kernel|cols_kernel|l2t_warp|s2m_warp" -c 4 -o gpurun_out/c4_far_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_far.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_dense -s 2 -c 1 -o gpurun_out/m2l_dense_B64 python tools/m2l_ab.py > gpurun_out/ncu_m2l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rows|cols" -c 2 -o gpurun_out/interp_B64 python tools/rs_prof.py 64 > gpurun_out/ncu_rs64.log 2>&1
cat gpurun_out/pytest_gpu.log
tail -c 800 gpurun_out/bench.log
cat gpurun_out/bench_ref.log | tail -2
