cd $GRAFT_REPO_ROOT
CJM_LIB=build/var/libcjm_dyn.so timeout 300 python scripts/chunk_check.py
run() { CJM_LIB=build/var/libcjm_dyn.so timeout 300 python scripts/sweep_runner.py --warm 240 "$@" 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'], 'K', d['temporal_k'], 'chunk', d['chunk_rows'], 'w', d['warps'], round(d['us_per_sweep'],2), round(d['glups'],1))"; }
for K in 3 4; do for ch in -1 64 96 128 192 256; do run --config cjm9_4096 --count 2400 --variant 7 --temporal-k $K --chunk-rows $ch; done; done
for ch in -1 128 256 512; do run --config cjm9_16384 --count 400 --variant 7 --temporal-k 4 --chunk-rows $ch; done
