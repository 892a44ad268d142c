# A/B of library builds on the same box: per-sweep time, CFGS = "variant:K ..."
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for rep in 1 2; do
for lib in ${LIBS:-build/var/libcjm_old.so paper_1705_00103_b200/libcjm.so}; do
  for cfg in ${CFGS:-4:2 4:1 4:3 7:3 6:2}; do
    v=${cfg%%:*}; k=${cfg##*:}
    CJM_LIB=$lib timeout 300 python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count ${COUNT:-2400} --warm 240 --variant $v --temporal-k $k | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['config'], d['variant'], d['temporal_k'], round(d['us_per_sweep'],2), round(d['glups'],1))"
  done
done
done
