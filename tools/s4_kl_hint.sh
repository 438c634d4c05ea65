#!/bin/bash
# session 4: k_large L2 evict_last hints on the activation scratch.  cfg5 parity, interleaved A/B
# against libmlpv_prev.so, then the DRAM bytes per launch of both builds (ncu, two metrics only).
O=gpurun_out/$1; mkdir -p $O
STEPS=10 bash tools/r3_ab5.sh $1
for L in libmlpv.so libmlpv_prev.so; do
  MLPV_LIB=$PWD/paper_1907_12933_b200/$L timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_large -s 3 -c 1 --csv --log-file $O/dram_$L.csv python bench.py --config cfg5_bf16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_$L.log 2>&1
  echo "$L"; grep -E "dram__|gpu__time" $O/dram_$L.csv | cut -d, -f12-
done
