mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/bench_check.log 2>&1
cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_check.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["gpu_launches"], d["roofline"]["frac"], d["stages_ms"], d["setup_s"])
PY
