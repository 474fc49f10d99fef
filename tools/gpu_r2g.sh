# new rs2 / box2 instantiations (accuracy-policy grids): parity + C3_acc / C5_acc timing;
# per-direction launch bounds of the register-resident passes: A/B on C2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "grid_pairs or acc" > gpurun_out/r2g_pytest.log 2>&1
tail -3 gpurun_out/r2g_pytest.log
L=$PWD/paper_0911_4114_b200
: > gpurun_out/rs2minb.log
for r in 1 2; do
for v in "" dn3 uprows4; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 600 python tools/ops_ab.py 32 64 >> gpurun_out/rs2minb.log 2>&1
done; done
cat gpurun_out/rs2minb.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3_acc,C5_acc > gpurun_out/bench_acc.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/bench_acc.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("C4", d["ms_per_step"])
        for k, v in d.get("other_configs", {}).items():
            print(k, v["ms_per_matvec"], v["parity"]["rel_l2_vs_oracle"], v["parity"]["err_vs_direct"])
PY
