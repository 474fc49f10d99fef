#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/m2l_l1pf_ab.txt
: > $out
echo "[l1pf parity] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_l1pf.so timeout 900 python -m pytest tests/test_gpu_c2.py -k m2l -q 2>&1 | tail -1)" >> $out
for rep in 1 2; do
  for v in "" l1pf; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib python -c 'import sys, json; sys.path.insert(0, "."); import bench; d = bench.bench_operators([16, 32, 64], reps=3); print(json.dumps({B: round(d[B]["m2l"]["ms"], 3) for B in ("B16", "B32", "B64")}), json.dumps({B: round(d[B]["m2l"]["frac_fp64"], 3) for B in ("B16", "B32", "B64")}))' > gpurun_out/m2l_l1pf_$v.log 2>&1
    echo "${v:-default} $(tail -1 gpurun_out/m2l_l1pf_$v.log)" >> $out
  done
done
cat $out
