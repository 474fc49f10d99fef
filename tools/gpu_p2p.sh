mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/bench_v3.log 2>&1
HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_minb5.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/bench_v3_minb5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for f in ["gpurun_out/bench_v3.log", "gpurun_out/bench_v3_minb5.log"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["frac"], d["stages_ms"])
    except Exception as e:
        print(f, "ERR", e, open(f).read()[-2000:])
PY
