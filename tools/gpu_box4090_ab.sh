mkdir -p gpurun_out
HFMM_BOX2_4090=0 timeout 900 python -m pytest tests/test_gpu_baseline_parity.py -x -q -k "grid_pairs or acc" > gpurun_out/b4090_pytest.log 2>&1; tail -1 gpurun_out/b4090_pytest.log
: > gpurun_out/b4090_ab.jsonl
for r in 1 2; do for v in 1 0; do
  echo "{\"box2_4090\": $v}" >> gpurun_out/b4090_ab.jsonl
  HFMM_BOX2_4090=$v timeout 600 python tools/c5acc_stages.py C5 acc serial >> gpurun_out/b4090_ab.jsonl 2>&1
  HFMM_BOX2_4090=$v timeout 600 python tools/c5acc_stages.py C5 acc >> gpurun_out/b4090_ab.jsonl 2>&1
  HFMM_BOX2_4090=$v timeout 600 python tools/c5acc_stages.py C3 acc >> gpurun_out/b4090_ab.jsonl 2>&1
done; done
python - <<'PY'
import json
tag = None
for l in open("gpurun_out/b4090_ab.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l)
    if "box2_4090" in d: tag = d["box2_4090"]; continue
    st = d["stages_ms"]
    print("box2_4090=%s %s acc=%s serial=%s m2m %.2f l2l %.2f total %.2f" % (tag, d["config"], d["acc"], d["serial"], st["m2m"], st["l2l"], st["total"]))
PY
