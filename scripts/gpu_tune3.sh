# per-config comparison of the sweep-kernel variants (one line per run)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
run() { timeout 300 python scripts/sweep_runner.py --count ${COUNT:-2400} --warm 240 "$@" 2>&1 | tail -1; }
{
for cfg in cjm9_16384 cjm9_1024 cjm5_1024; do
  run --config $cfg --variant 4 --temporal-k 2 --stages 8
  run --config $cfg --variant 7 --temporal-k 3 --stages 6
  run --config $cfg --variant 7 --temporal-k 4 --stages 6
  run --config $cfg --variant 5 --temporal-k 4 --stages 8
done
run --config cjm17_8192 --variant 3 --temporal-k 1 --tile-w 512
run --config cjm17_8192 --variant 4 --temporal-k 1
for st in 3 4 6; do
  run --config cjm17_8192 --variant 6 --temporal-k 1 --stages $st
  run --config cjm17_8192 --variant 7 --temporal-k 1 --stages $st
  run --config cjm17_8192 --variant 7 --temporal-k 2 --stages $st
done
run --config cjm17_8192 --variant 5 --temporal-k 2 --stages 8
} > gpurun_out/tune3.log
python - <<PY
import json
for l in open('gpurun_out/tune3.log'):
    if not l.startswith('{'): print(l.rstrip()[:200]); continue
    r=json.loads(l)
    print(r['config'], r['variant'], r['temporal_k'], r['stages'], r.get('tile_w'), round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
