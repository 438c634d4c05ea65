#!/bin/bash
# session 4: does the nvidia-smi sampler running beside the timed steps slow them?  (e2e, measured
# after the sampler has stopped, is consistently a few % above the device-timed value)
O=gpurun_out/$1; mkdir -p $O
for i in 1 2 3; do for M in off 200 100 1000; do
  if [ $M = off ]; then export MLPV_BENCH_SAMPLER=off; else unset MLPV_BENCH_SAMPLER; export MLPV_BENCH_SAMPLER_MS=$M; fi
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('sampler=$M', 'value %.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], 'frac %.4f' % d['roofline']['frac'], 'kernel_ms %.3f' % d['roofline']['kernel_ms'], d['clocks'])"
done; done | tee $O/ab.txt
