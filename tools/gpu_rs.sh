# resample kernels: parity (C2 ops + matvec parity) and C2 operator + C4 timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c2.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/rs_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra "" > gpurun_out/rs_bench.log 2>&1
cat gpurun_out/rs_pytest.log
python - <<'PY'
import json
d = json.loads(open("gpurun_out/rs_bench.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["gpu_launches"], {k: round(v, 2) for k, v in d["stages_ms"].items()})
for B, r in d["operators"].items():
    if B.startswith("B"):
        print(B, {k: (round(v["ms"], 3), round(v["frac_hbm"], 3), round(v.get("frac_fp64", 0), 3)) for k, v in r.items()})
PY
