import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_00103_b200 import cjm, inputs
st, n, var, K, cnt = [int(x) for x in sys.argv[1:6]]
r = 2 if st == 17 else 1
u0, b, h = inputs.test_problem(n, n, r, init="random")
bd = torch.from_numpy(b).cuda()
ref_plan = cjm.Plan(st, n, n, h, 1e-8, temporal_k=1, variant=3)
plan = cjm.Plan(st, n, n, h, 1e-8, temporal_k=K, variant=var)
bad = 0
for t in range(int(sys.argv[6])):
    ua = torch.from_numpy(u0.copy()).cuda(); ub = ua.clone()
    ref_plan.sweeps(bd, ua, t, cnt); plan.sweeps(bd, ub, t, cnt)
    A, B = ua.cpu().numpy(), ub.cpu().numpy()
    if not np.array_equal(A, B):
        bad += 1
        d = np.argwhere(A != B)
        if bad <= 5:
            print("trial", t, "ndiff", len(d), "rows", sorted(set(d[:, 0]))[:10], "cols", sorted(set(d[:, 1]))[:10], flush=True)
print("bad", bad, flush=True)
