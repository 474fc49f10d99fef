# P2P variant parity (tile x row-skip) + three driver-style bench runs for run-to-run spread
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k p2p_tiles > gpurun_out/p2pvar_pytest.log 2>&1; tail -1 gpurun_out/p2pvar_pytest.log
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu-baseline --ops "" --extra "C3,C5_acc" > gpurun_out/bench_rep$i.log 2>&1
  python - $i <<'PY'
import json, sys
for l in open(f"gpurun_out/bench_rep{sys.argv[1]}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("rep", sys.argv[1], "C4 %.3f ms %.3f matvec/s e2e %.3f frac %.4f" % (d["ms_per_step"], d["value"], d["e2e"]["value"], d["roofline"]["frac"]),
              " ".join("%s %.3f" % (k, v["ms_per_matvec"]) for k, v in d.get("other_configs", {}).items()), d.get("clocks"))
PY
done
