# ncu --set full with source of the default 9-point sweep kernel at 4096^2 for
# K = 1 and K = 2 (each command first exits 0 without ncu)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-src}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for K in ${KS:-1 2}; do
SW="python scripts/sweep_runner.py --config cjm9_4096 --count 40 --temporal-k $K --variant ${VAR:-4}"
timeout 300 $SW > gpurun_out/plain_${TAG}_k$K.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cjm_sweep_kernel -s 8 -c 1 \
    -o gpurun_out/prof_${TAG}_k$K -f $SW > gpurun_out/ncu_${TAG}_k$K.log 2>&1; echo k${K}_ncu_exit=$?
done
