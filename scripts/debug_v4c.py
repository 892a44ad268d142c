import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_1705_00103_b200 import cjm, inputs
st, n, cnt, trials = [int(x) for x in sys.argv[1:5]]
r = 2 if st == 17 else 1
u0, b, h = inputs.test_problem(n, n, r, init="random")
bd = torch.from_numpy(b).cuda()
s = oracle.schedule(st, n, n, 1e-8)
g = oracle.rhs_to_g(st, h, b)
for var, K, stg in [(3, 1, 4), (3, 2, 4), (4, 1, 4), (4, 2, 4), (4, 1, 8), (4, 1, 2)]:
    plan = cjm.Plan(st, n, n, h, 1e-8, temporal_k=K, variant=var, stages=stg)
    bad = 0
    for t in range(trials):
        ref = oracle.sweeps(st, u0, g, s["w"], t, cnt) if t < 3 else None
        if t == 0: ref0 = {}
        ub = torch.from_numpy(u0.copy()).cuda()
        plan.sweeps(bd, ub, 0, cnt)
        B = ub.cpu().numpy()
        if t == 0:
            R0 = oracle.sweeps(st, u0, g, s["w"], 0, cnt)
        if not np.array_equal(R0, B):
            bad += 1
    print("variant", var, "K", K, "stages", stg, "bad", bad, "of", trials, flush=True)
    plan.close()
