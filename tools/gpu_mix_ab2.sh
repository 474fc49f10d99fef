#!/bin/bash
# Mixed P2P tiles, second same-box A/B: item order by padded slots (default) vs live pairs
# (HFMM_P2P_SORT=0), and the 384-point class cost of the tile cut (HFMM_P2P_MIX3COST 1.0 / 1.2 vs 1.08).
mkdir -p gpurun_out
out=gpurun_out/mix_ab2.txt
: > $out
for rep in 1 2; do
  for v in default sort0 cost100 cost120; do
    env=""
    [ "$v" = "sort0" ] && env="HFMM_P2P_SORT=0"
    [ "$v" = "cost100" ] && env="HFMM_P2P_MIX3COST=1.0"
    [ "$v" = "cost120" ] && env="HFMM_P2P_MIX3COST=1.2"
    env $env timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5 > gpurun_out/mixab2_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/mixab2_{v}.log").read().strip().splitlines()[-1])
    oc = d["other_configs"]
    print(v, "C4", round(d["ms_per_step"], 2), "p2p", round(d["roofline"]["launch_ms"], 2), "serial", round(d["roofline"]["launch_ms_serial"], 2), "frac", round(d["roofline"]["frac"], 3), "mixed items", d["plan"].get("p2p_mixed_items"), "parity", d["parity"].get("rel_l2_vs_oracle"), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1), "C5 mixed", oc["C5"].get("p2p_mixed_items"))
except Exception as e:
    print(v, "FAILED", e)
PY
  done
done
cat $out
