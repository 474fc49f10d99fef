# plan-level row skipping: threshold A/B (off / default 8% / always) and kernel flavour (mode 1 / 2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p or direct or matvec" > gpurun_out/rowskip2_pytest.log 2>&1; tail -2 gpurun_out/rowskip2_pytest.log
HFMM_P2P_ROWSKIP_MIN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p2p or direct or matvec" >> gpurun_out/rowskip2_pytest.log 2>&1; tail -2 gpurun_out/rowskip2_pytest.log
L=$PWD/paper_0911_4114_b200
: > gpurun_out/rowskip_ab2.log
for r in 1 2; do
for v in "off::1.0" "def::0.08" "on::0.0" "m2on:rsmode2:0.0"; do
  tag=${v%%:*}; rest=${v#*:}; lv=${rest%%:*}; thr=${rest#*:}
  lib=""; [ -n "$lv" ] && lib="$L/libhfmm_$lv.so"
  HFMM_LIB=$lib HFMM_P2P_ROWSKIP_MIN=$thr timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5,C3_acc,C5_acc > gpurun_out/rowskip_b2.log 2>&1
  python - "$tag" >> gpurun_out/rowskip_ab2.log <<'PY'
import json, sys
for l in open("gpurun_out/rowskip_b2.log"):
    if l.startswith("{"):
        d = json.loads(l)
        oc = d.get("other_configs", {})
        pl = d["plan"]
        print(sys.argv[1], "C4 %.3f (rs %d dead %.3f)" % (d["ms_per_step"], pl["p2p_rowskip"], pl["p2p_dead_frac"]),
              " ".join("%s %.3f (t%d rs %d dead %.3f)" % (k, v["ms_per_matvec"], v["p2p_tile"], v["p2p_rowskip"], v["p2p_dead_frac"]) for k, v in oc.items()))
PY
done; done
cat gpurun_out/rowskip_ab2.log
