#!/bin/bash
# quick k_large check: build, cfg5 parity tests, traces, bench lines
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_parity_large_gpu.py -x -q -m gpu ${PYK:+-k "$PYK"} > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for c in cfg5_bf16 cfg5_int8; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; tail -1 $O/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])"
done
python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1
for c in cfg5_bf16 cfg5_int8; do timeout 200 python tools/trace_large.py $c 4096 > $O/trace_$c.txt 2>&1; sed -n 3p $O/trace_$c.txt; tail -6 $O/trace_$c.txt | cut -c1-250; done
