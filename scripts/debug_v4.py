import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_00103_b200 import cjm, inputs
st, n = int(sys.argv[1]), int(sys.argv[2])
r = 2 if st == 17 else 1
u0, b, h = inputs.test_problem(n, n, r)
bd = torch.from_numpy(b).cuda()
P = cjm.cjm_schedule(st, n, n, 1e-8)["P"]
print("P", P)
for first, count in [(0, 1), (0, 2), (0, 64), (0, 65), (1, 64), (1, 6560), (0, 6561), (0, P + 3)]:
    outs = []
    for var in (3, 4):
        for K in (1, 2):
            with cjm.Plan(st, n, n, h, 1e-8, temporal_k=K, variant=var) as plan:
                ud = torch.from_numpy(u0.copy()).cuda()
                plan.sweeps(bd, ud, first, count)
                outs.append(((var, K), ud.cpu().numpy()))
    ref = outs[0][1]
    print(first, count, [(k, bool(np.array_equal(o, ref)), float(np.max(np.abs(o - ref)))) for k, o in outs], flush=True)
