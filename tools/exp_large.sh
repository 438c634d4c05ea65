#!/bin/bash
# k_large timing experiments: product build vs MLPV_EXP variants (results wrong by design)
python -m paper_1907_12933_b200.build > /dev/null 2>&1 || exit 1
for X in ${EXPS:-201 202}; do
  MLPV_EXP=$X python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1 || exit 1
  cp paper_1907_12933_b200/libmlpv_trace.so paper_1907_12933_b200/libmlpv_exp$X.so
done
for c in ${CFGS:-cfg5_bf16 cfg5_int8}; do for L in libmlpv.so $(for X in ${EXPS:-201 202}; do echo libmlpv_exp$X.so; done); do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"kernel_ms\": [0-9.]*" | tr "\n" " "; echo " $c $L"
done; done
