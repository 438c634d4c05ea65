#!/bin/bash
# compute-sanitizer runs (memcheck, racecheck, synccheck) on small slices; logs under gpurun_out/TAG
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for c in cfg2 cfg4 cfg5_int8 cfg5_bf16; do
    timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_run.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/${tool}_$c.log | tail -1)"
  done
done
