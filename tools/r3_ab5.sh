#!/bin/bash
# k_large A/B: cfg5 parity tests on the new build, then interleaved cfg5 bf16 / int8 bench runs of
# libmlpv.so vs libmlpv_prev.so.  usage: tools/r3_ab5.sh TAG
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_large_gpu.py -q -x -k "cfg5 or int8 or restriction" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for c in cfg5_int8 cfg5_bf16; do for i in 1 2 3; do for L in libmlpv.so libmlpv_prev.so; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*\|\"frac\": [0-9.]*" | tr "\n" " "; echo " $c $L"
done; done; done | tee $O/ab.txt
