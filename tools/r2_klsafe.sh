#!/bin/bash
# k_large change check with a wait-timeout build first (a lost arrive traps instead of hanging)
O=gpurun_out/$1; mkdir -p $O
MLPV_WAIT_TIMEOUT=4000000000 python -m paper_1907_12933_b200.build --trace --force > $O/build_to.log 2>&1 || { tail $O/build_to.log; exit 1; }
MLPV_LIB=$PWD/paper_1907_12933_b200/libmlpv_trace.so timeout 300 python -m pytest tests/test_parity_large_gpu.py -x -q -m gpu > $O/pytest_to.log 2>&1
rc=$?; tail -15 $O/pytest_to.log; echo "timeout-build pytest rc=$rc"
[ $rc -eq 0 ] || exit 1
bash tools/r2_klq.sh $1
