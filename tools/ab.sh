#!/bin/bash
# A/B wall-clock comparison of the current build against paper_1907_12933_b200/libmlpv_prev.so
# (power-capped box: long runs, interleaved)
for i in 1 2; do for L in libmlpv.so libmlpv_prev.so; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*" | tr "\n" " "; echo " $L"
done; done
