cd $GRAFT_REPO_ROOT
TAG=${TAG:-s4}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-2500
timeout 900 python scripts/results_table.py > gpurun_out/results_${TAG}.jsonl 2>&1; echo rt_exit=$?
cut -c1-420 gpurun_out/results_${TAG}.jsonl
for cfg in cjm9_16384; do timeout 300 python scripts/sweep_runner.py --config $cfg --count 400 --warm 40 2>&1 | tail -1; done
