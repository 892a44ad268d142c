# GPU parity suite, then per-sweep times of every warp-tiled variant at 4096^2
cd $GRAFT_REPO_ROOT
TAG=${TAG:-t2}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
timeout 1500 python scripts/sweep_runner.py --tune --config ${CONFIG:-cjm9_4096} --ks ${KS:-1,2,3,4} --variants ${VARS:-4,5,6,7} \
   --stages-list ${STAGES:-3,4,6,8} --cps-list ${CPS:-2} > gpurun_out/tune_${TAG}.log 2>&1; echo tune_exit=$?
python - <<PY
import json
for l in open('gpurun_out/tune_${TAG}.log'):
    if not l.startswith('{'): continue
    r=json.loads(l)
    if 'glups' not in r: continue
    print(r['config'], r['variant'], r['temporal_k'], r['stages'], r['ctas_per_sm'], round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
