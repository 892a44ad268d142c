import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1705_00103_b200 import cjm, inputs
st, n = int(sys.argv[1]), int(sys.argv[2])
r = 2 if st == 17 else 1
u0, b, h = inputs.test_problem(n, n, r)
for var in (3, 4):
    for K in (1, 2):
        if st == 17 and var == 4 and K > 1: continue
        with cjm.Plan(st, n, n, h, 1e-8, temporal_k=K, variant=var) as plan:
            ud = torch.from_numpy(u0.copy()).cuda()
            rep = plan.solve(torch.from_numpy(b).cuda(), ud, ok=(0, 3, 4, 5))
            print(var, K, rep["status"], rep["iterations"], rep["cycles"], rep["r0_l2"], rep["r_l2"] / rep["r0_l2"], flush=True)
