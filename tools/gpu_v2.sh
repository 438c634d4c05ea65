#!/bin/bash
# first run of a new kernel: debug build (trap on lost arrivals) -> large parity tests -> normal build -> trace -> all gpu tests -> bench
O=gpurun_out/$1; mkdir -p $O
MLPV_WAIT_TIMEOUT=2000000000 python -m paper_1907_12933_b200.build --force > $O/build_dbg.log 2>&1 || exit 1
timeout 300 python -m pytest tests/test_parity_large_gpu.py -x -q > $O/large_dbg.log 2>&1; rc=$?; tail -5 $O/large_dbg.log
[ $rc -ne 0 ] && exit 1
python -m paper_1907_12933_b200.build --force > $O/build.log 2>&1 || exit 1
timeout 300 python tools/trace_fused3.py > $O/trace.log 2>&1; tail -14 $O/trace.log
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1; cat $O/bench.log
