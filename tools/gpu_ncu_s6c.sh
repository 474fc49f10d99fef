# session 6: full ncu capture of the <= 384-point P2P class (p2p_sym_kernel<0, 3, 4, 0>, second symmetric
# launch of a matvec) -- its counters came back empty as the second kernel of the first capture pass
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/s6c_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_sym_kernel -s 13 -c 1 \
  -o gpurun_out/s6c_p2p3 python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/s6c_ncu.log 2>&1
ncu -i gpurun_out/s6c_p2p3.ncu-rep --page details --csv > gpurun_out/ncu_full_p2p_sym3_s6_details.csv 2>/dev/null
ncu -i gpurun_out/s6c_p2p3.ncu-rep --page raw --csv > gpurun_out/ncu_full_p2p_sym3_s6_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import csv
rows = list(csv.DictReader(open("gpurun_out/ncu_full_p2p_sym3_s6_raw.csv")))
for r in rows[1:]:
    print(r["Kernel Name"][:60], r["gpu__time_duration.sum"], r["dram__bytes_read.sum"], r["dram__bytes_write.sum"], r["launch__grid_size"], r.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"))
print(rows[0]["gpu__time_duration.sum"], rows[0]["dram__bytes_read.sum"], rows[0]["dram__bytes_write.sum"])
PY
