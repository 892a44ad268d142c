cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python scripts/sweep_runner.py --tune --config ${TUNE_CFG:-cjm9_4096} --ks ${TUNE_KS:-1,2,3} --variants ${TUNE_VARS:-3,4} > gpurun_out/tune_${TAG:-x}.log 2>&1; echo tune_exit=$?
python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/tune_${TAG:-x}.log') if l.startswith('{')]
best={}
for r in rows:
    if 'glups' not in r: print(r); continue
    k=(r['config'],r.get('variant'),r['temporal_k'],r['tile_w'])
    if k not in best or r['glups']>best[k]['glups']: best[k]=r
for k,r in sorted(best.items()): print(k, r['stages'], r['ctas_per_sm'], round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
