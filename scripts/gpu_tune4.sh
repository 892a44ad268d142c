# variant 7: consumer warps per CTA x ring stages x K (one line per run), then auto
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
run() { timeout 300 python scripts/sweep_runner.py --warm 240 "$@" 2>&1 | tail -1; }
{
for K in 2 3 4; do for w in 4 5 7; do for st in 4 5 6; do
  run --config cjm9_4096 --count 2400 --variant 7 --temporal-k $K --warps $w --stages $st
done; done; done
for K in 3 4; do for w in 4 5 7; do
  run --config cjm9_16384 --count 400 --variant 7 --temporal-k $K --warps $w
done; done
for K in 1 2; do for w in 4 5 7; do for st in 3 4; do
  run --config cjm17_8192 --count 600 --variant 7 --temporal-k $K --warps $w --stages $st
done; done; done
for cfg in cjm9_4096 cjm9_16384 cjm17_8192 cjm9_1024 cjm5_1024; do run --config $cfg --count 600; done
} > gpurun_out/tune4.log
python - <<PY
import json
for l in open('gpurun_out/tune4.log'):
    if not l.startswith('{'): print(l.rstrip()[:160]); continue
    r=json.loads(l)
    print(r['config'], 'v',r['variant'], 'K',r['temporal_k'], 'w',r['warps'], 'st',r['stages'], 'ctas',r['ctas'], round(r['us_per_sweep'],1), round(r['glups'],1), round(r['gbs_per_launch']))
PY
