#!/bin/bash
# k_large experiments: trace timelines + kernel times of MLPV_EXP variants, and DRAM bytes per launch
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
for X in ${EXPS:-207 209}; do
  MLPV_EXP=$X python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1 || exit 1
  cp paper_1907_12933_b200/libmlpv_trace.so paper_1907_12933_b200/libmlpv_exp$X.so
done
for c in ${CFGS:-cfg5_bf16 cfg5_int8}; do for L in libmlpv.so $(for X in ${EXPS:-207 209}; do echo libmlpv_exp$X.so; done); do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"kernel_ms\": [0-9.]*" | tr "\n" " "; echo " $c $L"
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_large -s 3 -c 1 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__|gpu__time" 
done; done
for X in ${EXPS:-207 209}; do
  MLPV_EXP=$X python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1 || exit 1
  MLPV_EXP=$X timeout 300 python tools/trace_large.py cfg5_bf16 4096 2>&1 | tail -4 > $O/trace_bf16_$X.txt
done
