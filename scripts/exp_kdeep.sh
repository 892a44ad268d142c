#!/bin/bash
# Deeper temporal blocking for the 5/9-point (K = 5, 9 consumer warps; K = 6,
# 8 warps; one CTA per SM) against the default (K = 4, 11 warps): us per sweep
# (CUDA events) and a field digest after the same sweeps (bitwise A/B).
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
for CFG in cjm9_4096 cjm9_16384; do
  CNT=240; [ $CFG = cjm9_16384 ] && CNT=120
  python scripts/sweep_runner.py --config $CFG --count $CNT --warm 60 --digest
  for KW in "5 9" "6 8"; do set -- $KW
    CJM_LIB=build/libcjm_kdeep.so python scripts/sweep_runner.py --config $CFG --count $CNT --warm 60 --digest --temporal-k $1 --warps $2
  done
  python scripts/sweep_runner.py --config $CFG --count $CNT --warm 60 --digest
done
