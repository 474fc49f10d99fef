# session-6 validation (mixed P2P tiles): full GPU suite, smoke, driver-style bench; one-tile plan with the
# two item orders (why the mixed plan gains more than its padded slots); C4 launch list and full
# ncu captures of the two symmetric P2P classes (each ncu pass after the plain run exited 0)
mkdir -p gpurun_out
bash tools/gpu_final_r2.sh
: > gpurun_out/mix0_sort_ab.txt
for v in "HFMM_P2P_MIX=0 HFMM_P2P_SORT=0" "HFMM_P2P_MIX=0 HFMM_P2P_SORT=1" "HFMM_P2P_MIX=1 HFMM_P2P_SORT=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ops "" --extra "" > gpurun_out/mix0_sort.log 2>&1
  python - "$v" >> gpurun_out/mix0_sort_ab.txt <<'PY'
import json, sys
d = json.loads(open("gpurun_out/mix0_sort.log").read().strip().splitlines()[-1])
print(sys.argv[1], "C4", round(d["ms_per_step"], 2), "p2p", round(d["roofline"]["launch_ms"], 2), "serial", round(d["roofline"]["launch_ms_serial"], 2), "frac", round(d["roofline"]["frac"], 3))
PY
done
cat gpurun_out/mix0_sort_ab.txt
python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/s6_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_c4_s6.csv \
  python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/ncu_launch_s6.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4_s6.csv > gpurun_out/launches_c4_s6_summary.txt 2>&1
head -32 gpurun_out/launches_c4_s6_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_sym_kernel -s 12 -c 2 \
  -o gpurun_out/s6_p2p python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/s6_ncu_p2p.log 2>&1
ncu -i gpurun_out/s6_p2p.ncu-rep --page details --csv > gpurun_out/ncu_full_p2p_sym_s6_details.csv 2>/dev/null
ncu -i gpurun_out/s6_p2p.ncu-rep --page raw --csv > gpurun_out/ncu_full_p2p_sym_s6_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out/ | tail -15
