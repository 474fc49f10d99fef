# antipodal S2M / L2T kernels (default) vs the generic ones (libhfmm_noanti.so, HFMM_ANTIPODAL=0):
# parity subset with both libraries, then serial stage times of C4 / C3 / C5 (tau = eps/10), two alternations
mkdir -p gpurun_out
L=$PWD/paper_0911_4114_b200
for v in "" noanti; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  HFMM_LIB=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_parity.py -x -q \
    -k "small or deep or c4_small or fullsize_subset or c1hf or edge or single_level" > gpurun_out/anti_pytest_${v:-anti}.log 2>&1
  echo "${v:-anti}: $(tail -1 gpurun_out/anti_pytest_${v:-anti}.log)"
done
: > gpurun_out/anti_ab.log
for r in 1 2; do for v in "" noanti; do
  lib=""; [ -n "$v" ] && lib="$L/libhfmm_$v.so"
  echo "== ${v:-anti}" >> gpurun_out/anti_ab.log
  for c in "C4 x serial" "C3 x serial" "C5 acc serial" "C3 acc serial"; do
    HFMM_LIB=$lib timeout 300 python tools/c5acc_stages.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config'], d['acc'], {k: round(v,3) for k,v in d['stages_ms'].items()})" >> gpurun_out/anti_ab.log 2>&1
  done
done; done
cat gpurun_out/anti_ab.log
