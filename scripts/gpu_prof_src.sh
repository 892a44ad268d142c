# ncu --set full with source of one sweep-kernel launch (each command first exits 0 without ncu)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-src}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
SW="python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count 40 ${ARGS}"
timeout 300 $SW > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cjm_sweep_kernel -s 8 -c 1 \
    -o gpurun_out/prof_${TAG} -f $SW > gpurun_out/ncu_${TAG}.log 2>&1; echo ncu_exit=$?
