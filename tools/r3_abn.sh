#!/bin/bash
# A/B/C... of prebuilt libraries: fused-path parity tests on each, then interleaved bench runs.
# usage: LIBS="libmlpv.so libmlpv_b.so" tools/r3_abn.sh TAG [CFG]
O=gpurun_out/$1; mkdir -p $O
for L in $LIBS; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 900 python -m pytest tests/test_parity_large_gpu.py -q -x -k "cfg4 or fused3" > $O/pytest_$L.log 2>&1; echo "pytest $L rc=$?"; tail -1 $O/pytest_$L.log
done
for i in $(seq ${PAIRS:-3}); do for L in $LIBS; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config ${2:-cfg4} --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*\|\"frac\": [0-9.]*" | tr "\n" " "; echo " $L"
done; done | tee $O/ab.txt
