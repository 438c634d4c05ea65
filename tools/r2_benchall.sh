#!/bin/bash
# every config's bench line (default steps, cpu baseline + parity on the timed sample) and the cfg4
# profile evidence (launch list of the same command, one --set full capture of k_fused3)
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
for c in cfg4 cfg1 cfg2 cfg3 cfg5_bf16 cfg5_int8 cfg4_box; do
  timeout 600 python bench.py --config $c > $O/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 $O/bench_$c.log > $O/bench_$c.jsonl
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 \
  -o $O/prof_cfg4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo "full capture rc=$?"
python tools/ncu_summary.py $O/prof_cfg4.ncu-rep "cfg4 k_fused3 (1000 bases x 65536 PHILOX_CLAMP samples, one launch), r2" > $O/summary_cfg4.txt 2>&1
