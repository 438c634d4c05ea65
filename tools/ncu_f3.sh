#!/bin/bash
# GPU-box routine for profile evidence: plain bench (must exit 0) -> ncu launch list of the same
# command (cold-cache per-launch times) -> one ncu --set full capture (with source) of k_fused3.
# usage: tools/ncu_f3.sh TAG   (outputs under gpurun_out/TAG/)
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 || { tail $O/plain.log; exit 1; }
cat $O/plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_l.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 \
  -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo "full capture rc=$?"
