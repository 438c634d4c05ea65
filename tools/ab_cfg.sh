#!/bin/bash
# A/B of the current build vs paper_1907_12933_b200/libmlpv_prev.so on the configs in $CFGS
for c in ${CFGS:-cfg5_bf16 cfg5_int8}; do for L in libmlpv.so libmlpv_prev.so; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"frac\": [0-9.e-]*" | tr "\n" " "; echo " $c $L"
done; done
