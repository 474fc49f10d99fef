# full GPU suite + driver-style bench after the round-2 session-4 changes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2h.log 2>&1
tail -3 gpurun_out/pytest_gpu_r2h.log
timeout 900 python bench.py > gpurun_out/bench_r2h.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_r2h.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("C4", d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d.get("clocks"))
        for k, v in d.get("other_configs", {}).items():
            print(k, v["ms_per_matvec"], v.get("p2p_tile"), v["parity"]["rel_l2_vs_oracle"], v["parity"]["err_vs_direct"])
        for B in ("B8", "B16", "B32", "B64"):
            o = d.get("operators", {}).get(B)
            if o: print(B, {k: round(v["ms"], 3) for k, v in o.items()})
PY
