#!/bin/bash
# ncu evidence for cfg3's k_small on a 4 x 2^20 subset (the bench step is the whole 1.68e9 space)
O=gpurun_out/$1; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
timeout 120 python tools/small_run.py cfg3 4 1048576 3 > $O/plain.log 2>&1 || { tail $O/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_small} -s 2 -c 1 \
  -o $O/prof python tools/small_run.py cfg3 4 1048576 3 > $O/ncu_full.log 2>&1
echo "full capture rc=$?"
python tools/ncu_summary.py $O/prof.ncu-rep "cfg3 ${KREGEX:-k_small} (4 bases x 2^20)" > $O/summary.txt 2>&1; head -45 $O/summary.txt
