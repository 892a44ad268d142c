# v4 ring-slot release policies (CJM_V4_RELEASE 0..3): per-sweep time at
# 4096^2 for K = 1, 2, 3, then the ring stress test for the safe modes.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
cp paper_1705_00103_b200/libcjm.so build/var/libcjm_rel0.so
for m in 0 1 2 3; do
  for K in 1 2 3; do
    for r in 1 2; do
      CJM_LIB=build/var/libcjm_rel$m.so timeout 300 python scripts/sweep_runner.py --config cjm9_4096 --count 2400 --warm 240 --temporal-k $K --variant 4 | sed "s/^{/{\"mode\": $m, /"
    done
  done
done > gpurun_out/release_modes.jsonl 2>&1
cat gpurun_out/release_modes.jsonl | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['mode'], d['temporal_k'], round(d['us_per_sweep'],2), round(d['glups'],1), round(d['gbs_per_launch']))
    else: print(l.rstrip()[:200])"
for m in 1 2 3; do
  CJM_LIB=build/var/libcjm_rel$m.so timeout 600 python -m pytest tests/test_gpu_stress.py -q -x 2>&1 | tail -2 | sed "s/^/mode $m: /"
done
