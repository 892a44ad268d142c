set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python scripts/sweep_runner.py --tune --config cjm9_4096,cjm9_16384 > gpurun_out/tune.log 2>&1; echo tune_exit=$?
cat gpurun_out/tune.log | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin if l.startswith('{')]
for r in sorted(rows,key=lambda r:-r.get('gbs',0))[:12]: print(r)
"
timeout 300 python scripts/sweep_runner.py --config cjm9_4096 --count 30 > gpurun_out/plain_sweeps.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cjm_sweep_kernel -s 5 -c 3 -o gpurun_out/prof_sweep9_4096 python scripts/sweep_runner.py --config cjm9_4096 --count 30 > gpurun_out/ncu_full.log 2>&1; echo ncu_exit=$?
tail -3 gpurun_out/ncu_full.log
