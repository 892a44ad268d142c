import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.sweep_runner import run
for var, K in [(4, 2), (5, 2), (5, 3)]:
    for stg in (6, 8, 12, 16, 20, 24):
        for cps in (2, 3, 4):
            try:
                print(json.dumps(run("cjm9_4096", 2400, 240, variant=var, temporal_k=K, stages=stg, ctas_per_sm=cps)), flush=True)
            except Exception as e:
                print(json.dumps(dict(variant=var, K=K, stages=stg, cps=cps, error=str(e)[:80])), flush=True)
