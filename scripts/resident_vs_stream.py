import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1705_00103_b200 import cjm, inputs
for n in (64, 128, 256, 384, 512, 768, 1024):
    u0, b, h = inputs.test_problem(n, n, 1)
    bd = torch.from_numpy(b).cuda()
    row = {"n": n}
    for res in (1, -1):
        best = None
        try:
            for _ in range(3):
                ud = torch.from_numpy(u0.copy()).cuda()
                with cjm.Plan(9, n, n, h, 1e-8, resident=res) as plan:
                    rep = plan.solve(bd, ud)
                best = rep["solve_s"] if best is None else min(best, rep["solve_s"])
            row["res" if res == 1 else "stream"] = best * 1e3
            row["P"] = rep["cycle_len"]
        except cjm.CJMError as e:
            row["res" if res == 1 else "stream"] = str(e.name)
    print(json.dumps(row), flush=True)
