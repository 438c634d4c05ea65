#!/bin/bash
# cfg5 evidence for k_large after the CTA-pair rebuild: plain bench lines (must exit 0), the launch
# list of each command, one ncu --set full capture per variant, summaries; then the traced timelines.
# usage: tools/r2s3_kl.sh TAG
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
for c in cfg5_bf16 cfg5_int8; do
  timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_$c.log 2>&1 || { tail $O/plain_$c.log; exit 1; }
  tail -1 $O/plain_$c.log | cut -c1-300
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l_$c.log 2>&1
  echo "launch list $c rc=$?"
done
for c in cfg5_bf16 cfg5_int8; do
  timeout 300 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain1_$c.log 2>&1 || exit 1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_large -s 3 -c 1 \
    -o $O/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
  python tools/ncu_summary.py $O/prof_$c.ncu-rep "$c k_large (256 bases x 4096 samples, one launch), r2 CTA pairs" > $O/summary_$c.txt 2>&1
done
python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1
for c in cfg5_bf16 cfg5_int8; do timeout 200 python tools/trace_large.py $c 4096 > $O/trace_$c.txt 2>&1; done
python -m paper_1907_12933_b200.build --force > /dev/null 2>&1
