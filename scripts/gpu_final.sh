# Final checks of the round-1 kernel: smoke test, reference arm, 16384^2 and
# 17-point 8192^2 bench lines
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r01_v8}
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke_test_exit=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/smoke_${TAG}.log 2>&1; echo smoke_exit=$?
tail -3 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_${TAG}.log 2>&1; echo ref_exit=$?
tail -1 gpurun_out/ref_${TAG}.log | cut -c1-1500
timeout 900 python bench.py --config cjm9_16384 --steps 3 --warmup 3 > gpurun_out/bench16384_${TAG}.log 2>&1; echo b16384_exit=$?
tail -1 gpurun_out/bench16384_${TAG}.log | cut -c1-1500
timeout 600 python bench.py --config cjm17_8192 --steps 3 --warmup 3 > gpurun_out/bench17_${TAG}.log 2>&1; echo b17_exit=$?
tail -1 gpurun_out/bench17_${TAG}.log | cut -c1-1500
