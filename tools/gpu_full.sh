# Full round check: GPU tests, bench (with operators + cpu baseline), launch list, ncu captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader; nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_sym -s 3 -c 1 -o gpurun_out/p2p_sym_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"m2l_group|rows_kernel|cols_kernel" -c 3 -o gpurun_out/ops_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops 64 --extra "" > gpurun_out/ncu_ops.log 2>&1
cat gpurun_out/pytest_gpu.log
tail -c 800 gpurun_out/bench.log
cat gpurun_out/bench_ref.log | tail -2
