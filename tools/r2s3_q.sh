#!/bin/bash
# quick GPU check: build, the given pytest files, bench lines of the given configs (short).
# usage: PYT="tests/a.py tests/b.py" tools/r2s3_q.sh TAG CFG...
O=gpurun_out/$1; shift; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || { tail $O/build.log; exit 1; }
if [ -n "$PYT" ]; then timeout 1200 python -m pytest $PYT -q -x -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log; fi
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1
  tail -1 $O/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.4g' % d['value'], 'frac', round(d['roofline']['frac'], 4), 'kms', round(d['roofline']['kernel_ms'], 3), 'step', round(d['ms_per_step'], 3), 'mhz', d['clocks']['sm_mhz'], 'e2e %.4g' % d['e2e']['value'])" || tail -3 $O/bench_$c.log
done
