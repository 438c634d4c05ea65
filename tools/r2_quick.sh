#!/bin/bash
# quick k_fused3 iteration on the GPU box: bench cfg4 (x2, 20 steps) + the traced timeline.
# usage: tools/r2_quick.sh TAG [CFG]
O=gpurun_out/$1; C=${2:-cfg4}; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
python -m paper_1907_12933_b200.build --trace > $O/build_trace.log 2>&1 || exit 1
for i in 1 2; do
  timeout 300 python bench.py --config $C --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*\|\"frac\": [0-9.e-]*\|Error.*" | tr "\n" " "; echo " $C"
done > $O/ab.txt 2>&1
cat $O/ab.txt
timeout 600 python -m pytest tests/test_parity_large_gpu.py -q -x -k "cfg4 or fused3" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
MLPV_TRACE_CFG=$C timeout 300 python tools/trace_fused3.py > $O/trace.txt 2>&1
grep -E "period|E1 \(|E2 \(|E3 \(|gen rank 0|h1 wait" $O/trace.txt
