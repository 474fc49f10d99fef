#!/bin/bash
# Round-2 profiles (each ncu command only after its plain command exited 0):
#   1. the ncu launch list of the bench command (cold, serialised, clock-control none)
#   2. one full ncu capture of the dominant kernel (P2P symmetric, a timed-step launch)
#   3. full captures of the C2 B64 operators (interp rows2/cols2, m2l_dense) run alone
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --ops "" --extra "" > gpurun_out/r02_bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:p2p_sym_kernel -s 6 -c 1 \
  -o gpurun_out/r02_p2p_sym python bench.py --steps 1 --warmup 3 --ops "" --extra "" --no-cpu-baseline > gpurun_out/r02_ncu_p2p.log 2>&1
ncu -i gpurun_out/r02_p2p_sym.ncu-rep --page raw --csv > gpurun_out/r02_p2p_sym_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_p2p_sym.ncu-rep --page details --csv > gpurun_out/r02_p2p_sym_details.csv 2>/dev/null
ncu -i gpurun_out/r02_p2p_sym.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_p2p_sym_source_sass.csv 2>/dev/null
OPS='import sys; sys.path.insert(0, "."); import bench; print(bench.bench_operators([64], reps=1))'
python -c "$OPS" > gpurun_out/r02_ops_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"m2l_dense|rows2_kernel|cols2_kernel" -s 3 -c 5 \
  -o gpurun_out/r02_ops_b64 python -c "$OPS" > gpurun_out/r02_ncu_ops.log 2>&1
ncu -i gpurun_out/r02_ops_b64.ncu-rep --page raw --csv > gpurun_out/r02_ops_b64_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_ops_b64.ncu-rep --page details --csv > gpurun_out/r02_ops_b64_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
# deterministic near field: parity tests and the C4 cost
timeout 900 python -m pytest tests/test_gpu_parity.py -k deterministic -q > gpurun_out/r02_det_tests.log 2>&1
python - > gpurun_out/r02_det_ab.txt 2>&1 <<'PY'
import sys, time, statistics, json
sys.path.insert(0, ".")
import torch, numpy as np
import paper_0911_4114_b200 as hf
from workloads import CONFIGS, points_and_charges
cfg = CONFIGS["C4"]
x, q = points_and_charges(cfg)
qd = torch.from_numpy(q).cuda()
res = {}
for name, fl in (("atomic", 0), ("deterministic", hf.HFMM_DETERMINISTIC)):
    g = hf.HFMM(0); g.build_tree(x, cfg.depth, cfg.lo, cfg.size); g.precompute(cfg.kappa, cfg.eps, cfg.alpha, flags=fl)
    y = torch.empty_like(qd)
    for _ in range(3): g.matvec(qd, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(8):
        torch.cuda.synchronize(); e0.record(); g.matvec(qd, out=y); e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
    y1 = y.clone(); g.matvec(qd, out=y)
    res[name] = {"ms": statistics.mean(ms), "bitwise_repeat": bool(torch.equal(y1, y))}
    g.close()
print(json.dumps(res))
PY
cat gpurun_out/r02_det_tests.log | tail -2; cat gpurun_out/r02_det_ab.txt
ls -la gpurun_out | tail -20
