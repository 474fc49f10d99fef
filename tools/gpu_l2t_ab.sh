# L2T v3 (one warp reduction per point) vs v2 (reduction per 64 directions): parity + stage A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_virtual_ranks.py -x -q > gpurun_out/l2t_pytest.log 2>&1
tail -2 gpurun_out/l2t_pytest.log
timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "acc or subset or c4_small" >> gpurun_out/l2t_pytest.log 2>&1
tail -2 gpurun_out/l2t_pytest.log
L=$PWD/paper_0911_4114_b200
: > gpurun_out/l2t_ab.jsonl
for r in 1 2; do
for v in "" l2tv2 l2tpb8 oldlb; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  for a in "C5 acc serial" "C4 x serial" "C3 acc serial" "C3 x" "C3 x serial"; do
    echo "{\"lib\": \"$v\", \"args\": \"$a\"}" >> gpurun_out/l2t_ab.jsonl
    HFMM_LIB=$lib timeout 600 python tools/c5acc_stages.py $a >> gpurun_out/l2t_ab.jsonl 2>&1
  done
done; done
python - <<'PY'
import json
lib = None
for l in open("gpurun_out/l2t_ab.jsonl"):
    d = json.loads(l) if l.startswith("{") else None
    if d is None: print(l[:200]); continue
    if "lib" in d: lib = d["lib"] or "default(v3 pb4)"; continue
    st = d["stages_ms"]
    print(f"{lib:18s} {d['config']} acc={d['acc']} serial={d['serial']}  l2t {st['l2t']:.3f}  s2m {st['s2m']:.3f}  total {st['total']:.3f}")
PY
