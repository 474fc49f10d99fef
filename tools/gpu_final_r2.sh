# end-of-session validation: full GPU suite, smoke, driver-style bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -3 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_final.log"):
    if l.startswith("{"):
        d = json.loads(l)
        open("gpurun_out/bench_final.json", "w").write(l)
        print("C4", d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"], d.get("clocks"), d.get("gpu_launches"))
        for k, v in d.get("other_configs", {}).items():
            print(k, v["ms_per_matvec"], v.get("p2p_tile"), v.get("p2p_rowskip"), v["parity"]["rel_l2_vs_oracle"], v["parity"]["err_vs_direct"])
        for B in ("B8", "B16", "B32", "B64"):
            o = d.get("operators", {}).get(B)
            if o: print(B, {k: round(v["ms"], 3) for k, v in o.items()})
PY
