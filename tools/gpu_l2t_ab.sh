mkdir -p gpurun_out
: > gpurun_out/l2t_ab.log
echo "[l2tv2 parity] $(HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_l2tv2.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1)" >> gpurun_out/l2t_ab.log
for rep in 1 2; do
  for v in "" l2tv2; do
    lib=""; [ -n "$v" ] && lib="$PWD/paper_0911_4114_b200/libhfmm_$v.so"
    HFMM_LIB=$lib HFMM_PROFILE_STAGES=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" > gpurun_out/l2t_$v.log 2>&1
    python - "$v" >> gpurun_out/l2t_ab.log <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/l2t_{sys.argv[1]}.log").read().strip().splitlines()[-1])
oc = d.get("other_configs", {})
print(sys.argv[1] or "default", "C4", round(d["ms_per_step"], 2), "C3", round(oc["C3"]["ms_per_matvec"], 3), "C5", round(oc["C5"]["ms_per_matvec"], 1))
PY
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l2t -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops "" --extra "" 2>/dev/null | grep l2t | tail -2 >> gpurun_out/l2t_ab.log
HFMM_LIB=$PWD/paper_0911_4114_b200/libhfmm_l2tv2.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l2t -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --ops "" --extra "" 2>/dev/null | grep l2t | tail -2 >> gpurun_out/l2t_ab.log
cat gpurun_out/l2t_ab.log
