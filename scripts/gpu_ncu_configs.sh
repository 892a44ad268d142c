# One ncu --set full capture of the hot sweep kernel per large config (each
# command first exits 0 without ncu), for the bench line's traffic field
cd $GRAFT_REPO_ROOT
for cfg in cjm9_16384 cjm17_8192; do
SW="python scripts/sweep_runner.py --config $cfg --count 40"
timeout 300 $SW > gpurun_out/plain_sw_${cfg}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:cjm_sweep_kernel -s 4 -c 1 \
    -o gpurun_out/prof_r01_v8_${cfg} -f $SW > gpurun_out/ncu_full_${cfg}.log 2>&1; echo ${cfg}_ncu_exit=$?
tail -1 gpurun_out/ncu_full_${cfg}.log
done
