"""One default-plan solve of a bench config (for ncu captures of the check
launch: the solve's first sweep launch fuses the residual reduction).

    python scripts/one_solve.py [config]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIGS, make_problem  # noqa: E402
from paper_1705_00103_b200 import cjm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cjm9_4096"
st, nx, ny, tol = CONFIGS[cfg][:4]
u0, b, h = make_problem(st, nx, ny, 0, ny)
ud, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
with cjm.Plan(st, nx, ny, h, tol) as plan:
    rep = plan.solve(bd, ud)
print(json.dumps({k: rep[k] for k in ("status", "iterations", "temporal_k", "warps", "solve_s")}))
