mkdir -p gpurun_out
: > gpurun_out/p2p_ab.log
for v in t3m4; do
  echo "[$v parity] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1)" >> gpurun_out/p2p_ab.log
done
for rep in 1 2; do
  for v in "" t3m4 t4m3; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/p2pab_$v.log 2>&1
    python - "$v" >> gpurun_out/p2p_ab.log <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/p2pab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
oc = d.get("other_configs", {})
print(sys.argv[1] or "default", "C4", round(d["ms_per_step"], 2), "frac", round(d["roofline"]["frac"], 3), round(d["roofline"]["frac_serial"], 3), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1))
PY
  done
done
cat gpurun_out/p2p_ab.log
