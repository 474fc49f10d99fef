# session-5 validation: full GPU suite, smoke, driver-style bench, C4 launch list (ncu after the plain run)
mkdir -p gpurun_out
bash tools/gpu_final_r2.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_s5.csv \
  python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/ncu_launch_s5.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4_s5.csv 2>&1 | head -30
