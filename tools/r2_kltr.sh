#!/bin/bash
# k_large timelines (trace builds) of MLPV_EXP variants on cfg5_bf16: EXPS="201 203 206" tools/r2_kltr.sh TAG
O=gpurun_out/$1; mkdir -p $O
for X in ${EXPS:-201 203 206}; do
  MLPV_EXP=$X python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1 || exit 1
  MLPV_EXP=$X timeout 300 python tools/trace_large.py ${CFG:-cfg5_bf16} 4096 > $O/trace_$X.txt 2>&1
  sed -n 3p $O/trace_$X.txt; tail -4 $O/trace_$X.txt
done
