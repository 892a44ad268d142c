#!/bin/bash
# Interleaved A/B of library builds: sweep_runner (us per sweep, CUDA events;
# field digest for bitwise equality) for every build in LIBS on every config
# in CFGS, REPS times.  LIBS entries: "product" or a path to a measurement
# build.  Optional DIAG=<CJM_DIAG_TIMES build>: per-CTA busy fraction.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
LIBS=${LIBS:-product}
CFGS=${CFGS:-"cjm9_4096 cjm9_16384 cjm17_8192"}
for CFG in $CFGS; do
  CNT=240; [ $CFG = cjm9_16384 ] && CNT=120; [ $CFG = cjm17_8192 ] && CNT=120
  for REP in $(seq ${REPS:-2}); do
    for L in $LIBS; do
      if [ $L = product ]; then
        python scripts/sweep_runner.py --config $CFG --count $CNT --warm 60 --digest ${SWARGS}
      else
        CJM_LIB=$L python scripts/sweep_runner.py --config $CFG --count $CNT --warm 60 --digest ${SWARGS}
      fi
    done
  done
  if [ -n "$DIAG" ]; then CJM_LIB=$DIAG python scripts/diag_times.py $CFG; fi
done
