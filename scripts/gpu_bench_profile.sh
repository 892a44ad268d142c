# GPU parity suite, bench line, launch list, one full ncu capture of the hot
# sweep kernel (each ncu command first exits 0 without ncu)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo bench_exit=$?
tail -1 gpurun_out/bench_${TAG}.log | cut -c1-3000
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo launches_exit=$?
SW="python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count 40"
timeout 300 $SW > gpurun_out/plain_sw_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:cjm_sweep_kernel -s 4 -c 1 \
    -o gpurun_out/prof_${TAG} -f $SW > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu_full_exit=$?
tail -2 gpurun_out/ncu_full_${TAG}.log
