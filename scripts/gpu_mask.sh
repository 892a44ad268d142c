# generic-mask path (NEXT-4) on the GPU: mask parity tests, the rest of the
# GPU suite (unless SKIP_ALL), mask kernel measurement, ncu capture of the
# mask kernel (after the identical command exited 0 without ncu)
cd $GRAFT_REPO_ROOT
TAG=${TAG:-mask}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_masks.py -q -x > gpurun_out/pytest_masks_${TAG}.log 2>&1; echo masks_exit=$?
tail -15 gpurun_out/pytest_masks_${TAG}.log
if [ -z "$SKIP_ALL" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo pytest_exit=$?
tail -4 gpurun_out/pytest_gpu_${TAG}.log
fi
timeout 600 python scripts/mask_bench.py --tune > gpurun_out/mask_bench_${TAG}.log 2>&1; echo mask_bench_exit=$?
cut -c1-400 gpurun_out/mask_bench_${TAG}.log
timeout 300 python scripts/mask_bench.py --n 4096 --count 30 --solve-n 0 > gpurun_out/mask_small_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cjm_mask_kernel -s 40 -c 1 \
  -o gpurun_out/mask_full_${TAG} -f python scripts/mask_bench.py --n 4096 --count 30 --solve-n 0 \
  > gpurun_out/ncu_mask_${TAG}.log 2>&1; echo ncu_exit=$?
tail -3 gpurun_out/ncu_mask_${TAG}.log
