# launch lists (serialised, cold-cache per-launch durations) of the final round-2 library:
# the C4 bench command (driver recipe) and one C5 tau = eps/10 stage run
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_c4_r02f.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --ops "" --extra "" > gpurun_out/ncu_c4.log 2>&1
echo "c4 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c5acc_r02f.csv python tools/c5acc_stages.py C5 acc > gpurun_out/ncu_c5acc.log 2>&1
echo "c5acc rc=$?"
ls -la gpurun_out/launches_*r02f.csv
