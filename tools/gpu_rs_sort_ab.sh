# row-skipping plans (C3, C3/C5 at eps/10, C1-HF): items ordered by live rows x sources (default) vs live
# pairs (HFMM_P2P_SORT=0); then the new virtual-rank mixed-tile test and the tile parity tests
mkdir -p gpurun_out
out=gpurun_out/rs_sort_ab.txt
: > $out
for rep in 1 2; do
  for v in 1 0; do
    HFMM_P2P_SORT=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/rs_sort_$v.log 2>&1
    python - "$v" >> $out <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/rs_sort_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("HFMM_P2P_SORT=" + sys.argv[1], "C4", round(d["ms_per_step"], 2), " ".join(f"{k} {v['ms_per_matvec']:.3f}" for k, v in d["other_configs"].items()))
PY
  done
done
cat $out
timeout 900 python -m pytest tests/test_gpu_virtual_ranks.py tests/test_gpu_parity.py -x -q -k "mixed or tiles_agree" 2>&1 | tail -2
