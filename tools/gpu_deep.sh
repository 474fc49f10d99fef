mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/bench_deep.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_deep.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for f in ["gpurun_out/bench_deep.log"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["frac"], d["stages_ms"], d["plan"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-3000:])
PY
