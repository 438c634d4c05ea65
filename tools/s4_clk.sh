#!/bin/bash
# session 4: every config's clocks object with the in-process NVML sampler (and cfg4 with nvidia-smi)
O=gpurun_out/$1; mkdir -p $O
for c in cfg4 cfg1 cfg2 cfg3 cfg5_bf16 cfg5_int8 cfg4_box; do
  timeout 300 python bench.py --config $c --no-cpu-baseline 2>$O/err_$c.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c', '%.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], '%.4f' % d['roofline']['frac'], d['clocks'])"
done | tee $O/clk.txt
MLPV_BENCH_SAMPLER=smi timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('cfg4 smi', '%.4e' % d['value'], 'e2e %.4e' % d['e2e']['value'], '%.4f' % d['roofline']['frac'], d['clocks'])" | tee -a $O/clk.txt
