# Re-check the default launch shape of the 9-point kernel after the last
# kernel changes (4096^2 and 16384^2)
cd $GRAFT_REPO_ROOT
for cfg in cjm9_4096 cjm9_16384; do
  n=2400; [ $cfg = cjm9_16384 ] && n=400
  for opt in "" "--warps 5 --temporal-k 4" "--warps 5 --temporal-k 4 --ctas-per-sm 2" "--temporal-k 3" "--warps 11 --stages 8" "--warps 11 --stages 12"; do
    timeout 120 python scripts/sweep_runner.py --config $cfg --count $n --warm 200 $opt 2>&1 | tail -1 | cut -c1-400
  done
done
