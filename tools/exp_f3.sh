#!/bin/bash
# timing experiments of k_fused3 (trace build; results are wrong by design): MLPV_EXP=21 no generator
# stores, 104 weights only for tile 0, 105 no layer-3 MMAs, 106 E2 without TMEM loads / stores,
# 108 generators without Philox
for e in ${EXPS:-0 21 104}; do
  MLPV_EXP=$e python -m paper_1907_12933_b200.build --trace --force > /dev/null 2>&1
  echo "== MLPV_EXP=$e"; timeout 300 python tools/trace_fused3.py 2>&1 | grep -E "period|E1 \(|E2 \(|E3 \(|h1 wait|gen rank 0 grp 0|tile 10 stage-to-stage"
done
