#!/bin/bash
# round 3 (session 3) A/B: fused-path parity tests on the new build, then interleaved bench runs of
# libmlpv.so vs libmlpv_prev.so.  usage: tools/r3_ab.sh TAG [CFG]
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_parity_large_gpu.py tests/test_philox_gpu.py tests/test_parity_scale_gpu.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for i in 1 2 3; do for L in libmlpv.so libmlpv_prev.so; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 300 python bench.py --config ${2:-cfg4} --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*\|\"frac\": [0-9.]*" | tr "\n" " "; echo " $L"
done; done | tee $O/ab.txt
[ -n "$TRACE" ] && timeout 600 python tools/trace_fused3.py > $O/trace.txt 2>&1 && grep 'period\|E1 (\|E2 (' $O/trace.txt
