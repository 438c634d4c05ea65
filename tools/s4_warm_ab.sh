#!/bin/bash
# session 4: is the device-timed value lower than e2e because the first steps after a short warm-up
# see the power controller's transient?  interleaved bench runs with W = 3 / 20 / 40 (K = 5)
O=gpurun_out/$1; mkdir -p $O
for i in 1 2 3; do for W in 3 20 40; do
  timeout 300 python bench.py --no-cpu-baseline --warmup $W 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('W=$W', 'value %.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], d['clocks'])"
done; done | tee $O/ab.txt
