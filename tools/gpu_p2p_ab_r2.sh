#!/bin/bash
# P2P variant A/B (same box): default vs the variants given as arguments (libhfmm_<v>.so), parity
# of each variant first (small parity configs), then C4 / C3 / C5 matvec times.
mkdir -p gpurun_out
out=gpurun_out/p2p_ab_r2.txt
: > $out
for v in "$@"; do
  echo "[$v parity] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k 'small or deep or cube or c1' 2>&1 | tail -1)" >> $out
done
for rep in 1 2; do
  for v in "" "$@"; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra C3,C5 > gpurun_out/p2pab_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/p2pab_{v}.log").read().strip().splitlines()[-1])
oc = d["other_configs"]
print(v or "default", "C4", round(d["ms_per_step"], 2), "p2p", round(d["roofline"]["launch_ms"], 2), "serial", round(d["roofline"]["launch_ms_serial"], 2), "frac", round(d["roofline"]["frac"], 3), "parity", d["parity"].get("rel_l2_vs_oracle"), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1))
PY
  done
done
cat $out
