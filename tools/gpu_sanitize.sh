#!/bin/bash
# compute-sanitizer passes over the library's kernels (after a clean plain run): memcheck on the
# smoke matvecs, the small parity configs, the virtual ranks (R = 2) and the C2 B8 operators;
# racecheck (shared-memory hazards) and synccheck on the smoke matvecs and the B8 operators.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
out=gpurun_out/sanitize.txt
: > $out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_plain.log 2>&1; echo "plain smoke rc=$?" >> $out
run() {  # tool, name, command...
  local tool=$1 name=$2; shift 2
  timeout 1500 $CS --tool $tool --error-exitcode 99 --print-limit 20 "$@" > gpurun_out/san_${tool}_${name}.log 2>&1
  local rc=$?
  echo "$tool $name rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${name}.log | tail -1)" >> $out
}
run memcheck smoke python -c "import __graft_entry__ as g; g.smoke()"
run memcheck parity python -m pytest -x -q tests/test_gpu_parity.py -k "small or deep or cube or edge"
run memcheck vranks python -m pytest -x -q tests/test_gpu_virtual_ranks.py -k "2 and two_level"
run memcheck c2b8 python -m pytest -x -q tests/test_gpu_c2.py -k "8"
run racecheck smoke python -c "import __graft_entry__ as g; g.smoke()"
run racecheck c2b8 python -m pytest -x -q tests/test_gpu_c2.py -k "resample_ops and 8"
run synccheck smoke python -c "import __graft_entry__ as g; g.smoke()"
cat $out
