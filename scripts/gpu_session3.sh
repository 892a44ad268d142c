cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x > gpurun_out/pytest_slabs.log 2>&1; echo slabs_exit=$?; tail -2 gpurun_out/pytest_slabs.log
timeout 900 python scripts/fig4_right.py > gpurun_out/fig4_v7.log 2>&1; echo fig4_exit=$?
timeout 1200 python scripts/ratio_table.py > gpurun_out/ratios_v7.log 2>&1; echo ratios_exit=$?
run() { timeout 300 python scripts/sweep_runner.py --warm 120 --count 1200 "$@" 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'], 'v', d['variant'], 'K', d['temporal_k'], 'w', d['warps'], 'st', d['stages'], 'ctas', d['ctas'], 'ch', d.get('chunk_rows'), round(d['us_per_sweep'],2), round(d['glups'],1))"; }
for cfg in cjm9_1024 cjm5_1024 cjm17_1024; do
  run --config $cfg
  run --config $cfg --temporal-k 2
  run --config $cfg --temporal-k 1
  run --config $cfg --variant 4 --temporal-k 2
  run --config $cfg --temporal-k 3 --ctas-per-sm 1
  run --config $cfg --resident 1
done > gpurun_out/tune1024.log 2>&1
cat gpurun_out/tune1024.log
