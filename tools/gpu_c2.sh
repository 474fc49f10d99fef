mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_c2.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ops.log 2>&1
cat gpurun_out/pytest_c2.log; tail -c 3000 gpurun_out/bench_ops.log
