#!/bin/bash
# One parameterised GPU-session runner (replaces the round-1 one-off lease
# scripts).  Run under gpurun from the repo root:
#   gpurun --timeout 3000 -- 'TASKS="build tests bench ncu" TAG=r02 bash scripts/gpu_run.sh'
# TASKS (space-separated, run in order):
#   build     compile libcjm.so + oracle + build/fp64_peak (sm_100a)
#   tests     pytest -m gpu (the whole GPU suite) ; TESTS=<pytest args> narrows it
#   smoke     __graft_entry__.smoke()
#   bench     bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} --config ${CONFIG:-default}
#   ref       bench.py --impl reference (the oracle arm)
#   fp64      build/fp64_peak -> gpurun_out/fp64_peak_${TAG}.json
#   sweep     scripts/sweep_runner.py on ${CONFIG:-cjm9_4096} (${SWARGS})
#   launches  ncu launch list of a 1-step bench (after the same command exits 0)
#   ncu       ncu --set full of the hot sweep kernel via sweep_runner (after a plain run)
#   sanitize  compute-sanitizer --tool ${SANTOOL:-memcheck} on scripts/sanitize_cases.py
#   notma     the CJM_DIAG_NOTMA diagnostic build (producer issues no loads) timed by sweep_runner
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
TAG=${TAG:-run}
CONFIG_ARG=""
[ -n "$CONFIG" ] && CONFIG_ARG="--config $CONFIG"
for T in ${TASKS:-build tests}; do
  case $T in
    build)
      python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
      mkdir -p build && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak scripts/fp64_peak.cu
      echo build_exit=$? ;;
    tests)
      timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -x ${TESTS} > gpurun_out/pytest_gpu_${TAG}.log 2>&1
      echo pytest_exit=$?; tail -4 gpurun_out/pytest_gpu_${TAG}.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1
      echo smoke_exit=$?; tail -3 gpurun_out/smoke_${TAG}.log ;;
    bench)
      timeout ${BENCH_TIMEOUT:-1800} python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} $CONFIG_ARG ${BENCHARGS} \
        > gpurun_out/bench_${TAG}.log 2> gpurun_out/bench_${TAG}.err
      echo bench_exit=$?; tail -1 gpurun_out/bench_${TAG}.log | cut -c1-4000; tail -3 gpurun_out/bench_${TAG}.err ;;
    ref)
      timeout 1200 python bench.py --impl reference --steps ${STEPS:-3} --warmup ${WARMUP:-3} $CONFIG_ARG \
        > gpurun_out/ref_${TAG}.log 2>&1
      echo ref_exit=$?; tail -1 gpurun_out/ref_${TAG}.log | cut -c1-2000 ;;
    fp64)
      ./build/fp64_peak > gpurun_out/fp64_peak_${TAG}.json; echo fp64_exit=$?; cat gpurun_out/fp64_peak_${TAG}.json ;;
    sweep)
      timeout 600 python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count ${COUNT:-400} --warm 40 ${SWARGS} \
        > gpurun_out/sweep_${TAG}.log 2>&1; echo sweep_exit=$?; cat gpurun_out/sweep_${TAG}.log | tail -5 ;;
    launches)
      CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e $CONFIG_ARG"
      timeout 900 $CMD > gpurun_out/plain_launch_${TAG}.log 2>&1 && \
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-400} --csv \
        --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
      echo launches_exit=$? ;;
    ncu)
      SW="python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count 40 ${SWARGS}"
      timeout 300 $SW > gpurun_out/plain_sw_${TAG}.log 2>&1 && \
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cjm_sweep_kernel -s 6 -c ${NCU_COUNT:-1} \
        -o gpurun_out/prof_${TAG} -f $SW > gpurun_out/ncu_full_${TAG}.log 2>&1
      echo ncu_full_exit=$?; tail -2 gpurun_out/ncu_full_${TAG}.log ;;
    sanitize)
      timeout 300 python scripts/sanitize_cases.py > gpurun_out/plain_san_${TAG}.log 2>&1 && \
      timeout 2400 compute-sanitizer --tool ${SANTOOL:-memcheck} --error-exitcode 9 \
        python scripts/sanitize_cases.py > gpurun_out/sanitize_${SANTOOL:-memcheck}_${TAG}.log 2>&1
      echo sanitize_exit=$?; tail -4 gpurun_out/sanitize_${SANTOOL:-memcheck}_${TAG}.log ;;
    checked)
      # compute-sanitizer is closed on this pool: the CJM_DEBUG_CHECKS build
      # (device-side bounds checks of every TMA copy, ring read and store)
      # runs the GPU suite and the sanitizer cases; CJM_DEBUG_INJECT=1 is the
      # negative control that must be detected
      python -c "from paper_1705_00103_b200 import build as b; b.build(force=True, defines=('CJM_DEBUG_CHECKS',), out='build/libcjm_checked.so')" 2>&1 | tail -2
      CJM_LIB=build/libcjm_checked.so timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q ${TESTS} \
        > gpurun_out/pytest_checked_${TAG}.log 2>&1; echo checked_pytest_exit=$?; tail -3 gpurun_out/pytest_checked_${TAG}.log
      CJM_LIB=build/libcjm_checked.so timeout 600 python scripts/sanitize_cases.py > gpurun_out/checked_cases_${TAG}.log 2>&1
      echo checked_cases_exit=$?; tail -2 gpurun_out/checked_cases_${TAG}.log
      CJM_LIB=build/libcjm_checked.so CJM_DEBUG_INJECT=1 timeout 300 python scripts/sanitize_cases.py --inject \
        >> gpurun_out/checked_cases_${TAG}.log 2>&1; echo checked_inject_exit=$?; tail -1 gpurun_out/checked_cases_${TAG}.log ;;
    notma)
      python -c "from paper_1705_00103_b200 import build as b; b.build(force=True, defines=('CJM_DIAG_NOTMA',), out='build/libcjm_notma.so')" 2>&1 | tail -2
      for L in paper_1705_00103_b200/libcjm.so build/libcjm_notma.so; do
        CJM_LIB=$L timeout 600 python scripts/sweep_runner.py --config ${CONFIG:-cjm9_4096} --count 400 --warm 40 ${SWARGS}
      done > gpurun_out/notma_${TAG}.log 2>&1; echo notma_exit=$?; cat gpurun_out/notma_${TAG}.log ;;
    *) echo "unknown task $T" ;;
  esac
done
