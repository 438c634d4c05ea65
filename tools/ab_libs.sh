#!/bin/bash
# A/B of several prebuilt libraries on one config: LIBS="libmlpv.so libmlpv_x.so" CFG=cfg3 tools/ab_libs.sh
for i in 1 2; do for L in ${LIBS:-libmlpv.so libmlpv_prev.so}; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config ${CFG:-cfg4} --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*" | tr "\n" " "; echo " $L"
done; done
