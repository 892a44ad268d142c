# GPU suite, bench line, per-config sweep times of the defaults
cd $GRAFT_REPO_ROOT
TAG=${TAG:-s2}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-2500
for cfg in cjm9_4096 cjm9_16384 cjm17_8192 cjm9_1024 cjm5_1024 cjm17_1024; do
  timeout 300 python scripts/sweep_runner.py --config $cfg --count 400 --warm 40 2>&1 | tail -1
done > gpurun_out/defaults_${TAG}.jsonl
cat gpurun_out/defaults_${TAG}.jsonl | cut -c1-400
