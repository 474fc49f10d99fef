mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py tests/test_gpu_c2.py -x -q -k "grid_pairs or c2 or operator" > gpurun_out/r2i_pytest.log 2>&1
tail -2 gpurun_out/r2i_pytest.log
timeout 900 python bench.py > gpurun_out/bench_r2i.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_r2i.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("C4", d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d.get("clocks"), d.get("gpu_launches"))
        for k, v in d.get("other_configs", {}).items():
            print(k, v["ms_per_matvec"], v["parity"]["rel_l2_vs_oracle"], v["parity"]["err_vs_direct"])
        for B in ("B8", "B16", "B32", "B64"):
            o = d.get("operators", {}).get(B)
            if o: print(B, {k: round(v["ms"], 3) for k, v in o.items()})
        print("cpu_baseline", d.get("cpu_baseline"))
PY
timeout 300 python tools/c5acc_stages.py C5 acc >> gpurun_out/bench_r2i.log 2>&1; tail -1 gpurun_out/bench_r2i.log | cut -c1-400
