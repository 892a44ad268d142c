# tests + tuning + experiments in one GPU call (no ncu)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -4 gpurun_out/pytest_gpu_${TAG}.log
fi
if [ -n "$TUNE" ]; then
timeout 1200 python scripts/sweep_runner.py --tune --config ${TUNE_CFG:-cjm9_4096} --ks ${TUNE_KS:-1,2,3} --variants ${TUNE_VARS:-3,4} > gpurun_out/tune_${TAG}.log 2>&1; echo tune_exit=$?
python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/tune_${TAG}.log') if l.startswith('{')]
best={}
for r in rows:
    if 'glups' not in r: print(r); continue
    k=(r['config'],r.get('variant'),r['temporal_k'],r['tile_w'])
    if k not in best or r['glups']>best[k]['glups']: best[k]=r
for k,r in sorted(best.items()): print(k, r['stages'], r['ctas_per_sm'], round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
fi
if [ -n "$BENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-1500
fi
if [ -n "$EXPS" ]; then
timeout 900 python scripts/fig4_right.py > gpurun_out/fig4_${TAG}.log 2>&1; echo fig4_exit=$?
cat gpurun_out/fig4_${TAG}.log
timeout 1200 python scripts/ratio_table.py > gpurun_out/ratios_${TAG}.log 2>&1; echo ratios_exit=$?
cat gpurun_out/ratios_${TAG}.log | cut -c1-600
fi
