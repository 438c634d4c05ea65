#!/bin/bash
# every config's default bench line (cpu baseline + parity on the timed sample) -> gpurun_out/TAG/
O=gpurun_out/$1; mkdir -p $O
for c in cfg4 cfg1 cfg2 cfg3 cfg5_bf16 cfg5_int8 cfg4_box; do
  timeout 600 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 $O/bench_$c.log > $O/bench_$c.jsonl
done
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 $O/bench_ref.log > $O/bench_ref.jsonl
