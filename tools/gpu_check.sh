#!/bin/bash
# GPU-box routine: build, gpu tests, bench, launch list, one ncu --set full capture of the top kernel.
# usage: tools/gpu_check.sh [tag] [bench args...]
set -x
TAG=${1:-run}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py "$@" > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
