cd $GRAFT_REPO_ROOT
export CJM_LIB=build/var/libcjm_hyb.so
CJM_DYN_PCT=20 timeout 300 python scripts/chunk_check.py
CJM_DYN_PCT=100 timeout 300 python scripts/chunk_check.py
run() { timeout 300 python scripts/sweep_runner.py --warm 120 "$@" 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'], 'K', d['temporal_k'], 'w', d['warps'], 'ch', d.get('chunk_rows'), round(d['us_per_sweep'],2), round(d['glups'],1))"; }
for pct in 0 10 20 35 50 100; do for ch in 0 16 32 64; do
  echo -n "pct $pct "; CJM_DYN_PCT=$pct run --config cjm9_4096 --count 1200 --chunk-rows $ch
done; done
for pct in 0 20 50 100; do for ch in 0 64 128 256; do
  echo -n "pct $pct "; CJM_DYN_PCT=$pct run --config cjm9_16384 --count 200 --chunk-rows $ch
done; done
