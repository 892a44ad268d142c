# Run the CPU oracle for the large configs on the GPU box's host cores and
# bring the digests back in gpurun_out/oracle_digests.json (the box has more
# cores than the build container).  No GPU work.
cd $GRAFT_REPO_ROOT
python -c "import oracle; oracle.build(force=True); print('threads', oracle.num_threads())"
mkdir -p gpurun_out
cp tests/golden/oracle_digests.json gpurun_out/oracle_digests.json
CJM_DIGESTS_OUT=gpurun_out/oracle_digests.json timeout ${LIMIT:-7000} python tests/make_oracle_digests.py ${DIGESTS:-cjm17_8192 cjm9_16384} 2>&1 | tee gpurun_out/digests.log
echo digests_exit=$?
