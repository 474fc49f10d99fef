mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "grid_pairs or subset" > gpurun_out/c3cols_pytest.log 2>&1; tail -1 gpurun_out/c3cols_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c3_r02g.csv python tools/c5acc_stages.py C3 > gpurun_out/ncu_c3g.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3_r02g.csv | head -12
for i in 1 2; do timeout 300 python tools/c5acc_stages.py C3 | cut -c1-200; timeout 300 python tools/c5acc_stages.py C5 | cut -c1-200; done
