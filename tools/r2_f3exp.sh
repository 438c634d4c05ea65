#!/bin/bash
# k_fused3 clamp-vs-box comparison: bench A/B of cfg4 (PHILOX_CLAMP) and cfg4_box on one build, then
# the traced timelines of both.  usage: tools/r2_f3exp.sh TAG
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
for i in 1 2; do for c in cfg4 cfg4_box; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null \
    | grep -o "\"value\": [0-9.e+]*\|\"kernel_ms\": [0-9.]*\|\"sm_mhz\": [0-9.]*\|\"frac\": [0-9.e-]*" | tr "\n" " "; echo " $c"
done; done > $O/ab.txt 2>&1
cat $O/ab.txt
for c in cfg4 cfg4_box; do
  MLPV_TRACE_CFG=$c timeout 300 python tools/trace_fused3.py > $O/trace_$c.txt 2>&1
  grep -E "period|issuer per-stage|E1 \(|E2 \(|E3 \(|gen rank 0" $O/trace_$c.txt
done
