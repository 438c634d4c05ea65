#!/bin/bash
# interleaved 30-step runs of several builds: LIBS="libmlpv.so libX.so ..." (in paper_1907_12933_b200/)
for i in 1 2; do for L in ${LIBS}; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"sm_mhz\": [0-9.]*" | tr "\n" " "; echo " $L"
done; done
