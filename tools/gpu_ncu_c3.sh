mkdir -p gpurun_out
timeout 300 python tools/c5acc_stages.py C3 > gpurun_out/c3_plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c3_r02f.csv python tools/c5acc_stages.py C3 > gpurun_out/ncu_c3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3_r02f.csv
