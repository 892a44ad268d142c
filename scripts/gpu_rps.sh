# rows-per-stage variants (6, 7): GPU parity suite, then tuning at 4096^2
cd $GRAFT_REPO_ROOT
TAG=${TAG:-rps}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -4 gpurun_out/pytest_gpu_${TAG}.log
timeout 1500 python scripts/sweep_runner.py --tune --config cjm9_4096 --ks 1,2,3,4 --variants 6,7 \
   --stages-list 2,3,4,5,6 --cps-list 2,3,4 > gpurun_out/tune_${TAG}.log 2>&1; echo tune_exit=$?
timeout 600 python scripts/sweep_runner.py --tune --config cjm9_4096 --ks 1,2,3 --variants 4 \
   --stages-list 8 --cps-list 2 >> gpurun_out/tune_${TAG}.log 2>&1; echo tune4_exit=$?
python - <<PY
import json
for l in open('gpurun_out/tune_${TAG}.log'):
    if not l.startswith('{'): continue
    r=json.loads(l)
    if 'glups' not in r: print(r); continue
    print(r['variant'], r['temporal_k'], r['stages'], r['ctas_per_sm'], round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
