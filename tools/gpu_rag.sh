mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_rag.log
cat gpurun_out/pytest_rag.log
