"""Break down one bench step: cjm_plan, first/second cjm_solve, destroy."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS, make_problem  # noqa: E402
from paper_1705_00103_b200 import cjm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cjm9_4096"
st, nx, ny, tol = CONFIGS[cfg][:4]
u0, b, h = make_problem(st, nx, ny, 0, ny)
ud0, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
ud = ud0.clone()
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = cjm.Plan(st, nx, ny, h, tol)
    t1 = time.perf_counter()
    ud.copy_(ud0)
    r1 = plan.solve(bd, ud)
    t2 = time.perf_counter()
    ud.copy_(ud0)
    r2 = plan.solve(bd, ud)
    t3 = time.perf_counter()
    plan.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"plan {1e3*(t1-t0):.1f} ms (plan_s {1e3*r1['plan_s']:.1f}), solve1 {1e3*(t2-t1):.1f} ms "
          f"(dev {1e3*r1['solve_s']:.1f}, sweeps {1e3*r1['sweep_s']:.1f}, launches {r1['hot_launches']}), "
          f"solve2 {1e3*(t3-t2):.1f} ms (dev {1e3*r2['solve_s']:.1f}, sweeps {1e3*r2['sweep_s']:.1f}), "
          f"destroy {1e3*(t4-t3):.1f} ms", flush=True)
