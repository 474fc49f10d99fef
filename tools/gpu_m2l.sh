mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_m2l.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_m2l.log 2>&1
cat gpurun_out/pytest_m2l.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_m2l.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["gpu_launches"], d["stages_ms"])
for B, r in d["operators"].items():
    if B.startswith("B"):
        print(B, {k: (round(v["ms"], 3), round(v["frac_hbm"], 3), round(v.get("frac_fp64", 0), 3)) for k, v in r.items()})
PY
