# session-6 final validation (mixed tiles, row-skipping variants at 2x unrolling): full GPU suite, smoke,
# driver-style bench, reference arm (short), C4 launch list after the plain run
mkdir -p gpurun_out
bash tools/gpu_final_r2.sh
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference_s6.json 2> gpurun_out/bench_reference_s6.err; echo "reference exit $?"; head -c 600 gpurun_out/bench_reference_s6.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_c4_s6b.csv \
  python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/ncu_launch_s6b.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4_s6b.csv > gpurun_out/launches_c4_s6b_summary.txt 2>&1
head -8 gpurun_out/launches_c4_s6b_summary.txt
