#!/bin/bash
# cfg5 evidence for k_large: plain bench lines (must exit 0), then one ncu --set full capture per variant.
# usage: tools/ncu_large.sh TAG   (outputs under gpurun_out/TAG/)
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
for c in cfg5_bf16 cfg5_int8; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/$c.log 2>&1 || { tail $O/$c.log; exit 1; }
  tail -1 $O/$c.log
done
for c in cfg5_bf16 cfg5_int8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_large -s 3 -c 1 \
    -o $O/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"
done
