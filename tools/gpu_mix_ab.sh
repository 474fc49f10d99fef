#!/bin/bash
# Mixed P2P tiles + P2P instruction variants, same-box A/B: parity of the new plan first, then
# C4 / C3 / C5 matvec times for: default (mixed tiles on), mix0 (HFMM_P2P_MIX=0), and the variant
# libraries given as arguments (libhfmm_<v>.so, mixed tiles on).
mkdir -p gpurun_out
out=gpurun_out/mix_ab.txt
: > $out
echo "[mixed-tile parity] $(timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k 'mixed_tiles or tiles_agree or deterministic' 2>&1 | tail -1)" >> $out
for v in "$@"; do
  echo "[$v parity] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k 'mixed_tiles or small or deep' 2>&1 | tail -1)" >> $out
done
for rep in 1 2; do
  for v in "" mix0 "$@"; do
    lib=""; mix=1
    [ "$v" = "mix0" ] && mix=0
    [ -n "$v" ] && [ "$v" != "mix0" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_P2P_MIX=$mix HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5 > gpurun_out/mixab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/mixab_{v}.log").read().strip().splitlines()[-1])
    oc = d["other_configs"]
    print(v or "default", "C4", round(d["ms_per_step"], 2), "p2p", round(d["roofline"]["launch_ms"], 2), "serial", round(d["roofline"]["launch_ms_serial"], 2), "frac", round(d["roofline"]["frac"], 3), "launches", d["gpu_launches"], "parity", d["parity"].get("rel_l2_vs_oracle"), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1), "C5 parity", oc["C5"]["parity"].get("rel_l2_vs_oracle"))
except Exception as e:
    print(v or "default", "FAILED", e)
PY
  done
done
cat $out
