cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?
tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/sweep_runner.py --tune --config cjm9_4096 > gpurun_out/tune2.log 2>&1; echo tune_exit=$?
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/tune2.log') if l.startswith('{')]
for r in sorted(rows,key=lambda r:-r.get('glups',0))[:15]: print(r)
PY
