#!/bin/bash
# one ncu --set full capture (with source) of the top kernel of `bench.py --config CFG`, after the
# plain bench exits 0.  usage: tools/r2_ncu.sh TAG CFG KERNEL_REGEX
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
timeout 300 python bench.py --config $2 --steps 3 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 || { tail $O/plain.log; exit 1; }
tail -1 $O/plain.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 \
  -o $O/prof python bench.py --config $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo "full capture rc=$?"
python tools/ncu_summary.py $O/prof.ncu-rep "$2 $3" > $O/summary.txt 2>&1; cat $O/summary.txt
