#!/bin/bash
# session 4: does nvidia-smi's start-up inside the timed region slow the device-timed steps?
# interleaved bench runs, sampler started before the warm-up (default) vs at the timed region (late)
O=gpurun_out/$1; mkdir -p $O
for i in 1 2 3 4; do for M in early late; do
  MLPV_BENCH_SAMPLER=$M timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$M', 'value %.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], d['clocks'])"
done; done | tee $O/ab.txt
