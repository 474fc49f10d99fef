# symmetric P2P warp-row skipping: parity + same-box A/B on the matvec configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/rowskip_pytest.log 2>&1; tail -2 gpurun_out/rowskip_pytest.log
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "subset or acc or c4_small" >> gpurun_out/rowskip_pytest.log 2>&1; tail -2 gpurun_out/rowskip_pytest.log
L=$PWD/paper_0911_4114_b200
: > gpurun_out/rowskip_ab.log
for r in 1 2; do
for v in "" noskip; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5,C3_acc,C5_acc > gpurun_out/rowskip_b.log 2>&1
  python - "$v" >> gpurun_out/rowskip_ab.log <<'PY'
import json, sys
for l in open("gpurun_out/rowskip_b.log"):
    if l.startswith("{"):
        d = json.loads(l)
        oc = d.get("other_configs", {})
        print(sys.argv[1] or "rowskip", "C4 %.3f" % d["ms_per_step"], "frac %.4f" % d["roofline"]["frac"],
              " ".join("%s %.3f" % (k, v["ms_per_matvec"]) for k, v in oc.items()),
              "parity", " ".join("%s %.1e" % (k, v["parity"]["rel_l2_vs_oracle"]) for k, v in oc.items()))
PY
done; done
cat gpurun_out/rowskip_ab.log
