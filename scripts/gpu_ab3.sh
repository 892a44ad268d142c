# A/B: ABLIBS x (CFGS as variant:K) with extra sweep_runner args XARGS_<n>
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for cfg in ${CONFIGS:-cjm9_4096}; do
for lib in ${ABLIBS}; do
  for a in "${A1}" "${A2}" "${A3}" "${A4}"; do
    [ -z "$a" ] && continue
    CJM_LIB=$lib timeout 300 python scripts/sweep_runner.py --config $cfg --count ${COUNT:-1200} --warm 120 $a 2>&1 | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['config'], 'v', d['variant'], 'K', d['temporal_k'], 'w', d['warps'], 'st', d['stages'], 'ctas', d['ctas'], round(d['us_per_sweep'],2), round(d['glups'],1))" 2>&1 | tail -1
  done
done; done; done
