# full ncu capture of the hot sweep kernel for one launch configuration
cd $GRAFT_REPO_ROOT
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
SW="python scripts/sweep_runner.py --config ${CFG:-cjm9_4096} --count 40 ${SWARGS}"
timeout 300 $SW > gpurun_out/plain_sw_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cjm_sweep_kernel -s 6 -c 2 \
    -o gpurun_out/prof_${TAG} $SW > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu_full_exit=$?
cat gpurun_out/plain_sw_${TAG}.log
