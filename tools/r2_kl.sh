set -x
O=gpurun_out/r2kl; mkdir -p $O
python -m paper_1907_12933_b200.build > $O/build.log 2>&1 || exit 1
timeout 300 python tools/trace_large.py cfg5_bf16 4096 > $O/trace_bf16.txt 2>&1
timeout 300 python tools/trace_large.py cfg5_int8 4096 > $O/trace_int8.txt 2>&1
python -m paper_1907_12933_b200.build > $O/build2.log 2>&1 || exit 1
bash tools/r2_ncu.sh r2kl/ncu cfg5_bf16 k_large
