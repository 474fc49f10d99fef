#!/bin/bash
# P2P tile A/B (same box, same library): HFMM_P2P_PT forced to each value given vs the plan's
# choice; C4 / C3 / C5 matvec times and P2P stream time, two alternating repetitions.
mkdir -p gpurun_out
out=gpurun_out/pt_ab.txt
: > $out
for rep in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then unset HFMM_P2P_PT; else export HFMM_P2P_PT=$v; fi
    timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5 > gpurun_out/ptab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ptab_{v}.log").read().strip().splitlines()[-1])
oc = d["other_configs"]
print(v, "C4", round(d["ms_per_step"], 2), "p2p", round(d["roofline"]["launch_ms"], 2), "frac", round(d["roofline"]["frac"], 3), "parity", d["parity"].get("rel_l2_vs_oracle"), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1), "tile", d["plan"].get("p2p_tile"))
PY
  done
done
unset HFMM_P2P_PT
cat $out
