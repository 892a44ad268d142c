"""Small runs of every shipped kernel for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): the warp-tiled sweep kernel (one CTA of 11
consumer warps per SM at K = 4 with dynamic work items from the device
counter; the 17-point at K = 3; K = 1 remainder / residual launches), the
shared-line kernel (17-point K = 4), the shared-memory-resident cooperative
kernel, the check / reduction launches and the setup kernels, at 64^2 and
8192 x 64.  Each result is compared with the oracle, so a
run that the sanitizer slows down still has to be right.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1705_00103_b200 import cjm, inputs  # noqa: E402

CASES = [
    # (stencil, nx, ny, plan options, sweeps)
    (9, 64, 64, dict(resident=1), 12),
    (9, 64, 64, dict(resident=-1, temporal_k=4, warps=11, chunk_rows=4), 9),
    (9, 8192, 64, dict(temporal_k=4, warps=11, chunk_rows=4), 9),
    (9, 8192, 64, dict(), 7),
    (17, 8192, 64, dict(temporal_k=3, chunk_rows=4), 7),
    (17, 64, 64, dict(resident=-1, temporal_k=3), 7),
    (17, 300, 70, dict(temporal_k=4), 9),           # shared-line kernel (variant 3)
    (17, 64, 64, dict(resident=1), 8),
    (5, 8192, 64, dict(temporal_k=4, chunk_rows=4), 9),
]


def inject():
    """Negative control (CJM_DEBUG_CHECKS build with CJM_DEBUG_INJECT=1): the
    library understates the buffer size to the kernel, so its TMA bounds
    checks must fire and the call must fail."""
    u0, b, h = inputs.test_problem(300, 200, 1, init="random", seed=71)
    with cjm.Plan(9, 300, 200, h, 1e-8, resident=-1) as plan:
        try:
            plan.sweeps(torch.from_numpy(b).cuda(), torch.from_numpy(u0).cuda(), 0, 8)
        except cjm.CJMError as e:
            print("injected violation detected:", e)
            sys.exit(0)
    print("injected violation NOT detected")
    sys.exit(1)


def main():
    if "--inject" in sys.argv:
        inject()
    bad = 0
    for st, nx, ny, kw, cnt in CASES:
        r = oracle.reach(st)
        u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=71)
        with cjm.Plan(st, nx, ny, h, 1e-8, **kw) as plan:
            w = plan.info()["weights"]
            ud = torch.from_numpy(u0).cuda()
            rep = plan.sweeps(torch.from_numpy(b).cuda(), ud, 3, cnt)
            got = ud.cpu().numpy()
            l2, _ = plan.residual(torch.from_numpy(b).cuda(), torch.from_numpy(u0).cuda())
        want = oracle.sweeps(st, u0, oracle.rhs_to_g(st, h, b), w, 3, cnt)
        ok = np.array_equal(got, want)
        bad += not ok
        print(f"{st}-pt {nx}x{ny} {kw}: variant {rep['variant']} K={rep['temporal_k']} "
              f"warps={rep['warps']} resident={rep['resident']} bitwise={ok} r={l2:.3e}", flush=True)
    # one full solve (graphs, check launches, stop decision) per stencil at 64^2
    for st in (5, 9, 17):
        r = oracle.reach(st)
        u0, b, h = inputs.test_problem(64, 64, r)
        uo, ro = oracle.solve(st, h, 1e-8, b, u0)
        with cjm.Plan(st, 64, 64, h, 1e-8, resident=-1) as plan:
            ud = torch.from_numpy(u0).cuda()
            rep = plan.solve(torch.from_numpy(b).cuda(), ud)
        ok = rep["iterations"] == ro["iterations"] and np.array_equal(ud.cpu().numpy(), uo)
        bad += not ok
        print(f"{st}-pt 64^2 solve: {rep['status']} iterations={rep['iterations']} bitwise={ok}",
              flush=True)
    torch.cuda.synchronize()
    print("cases_failed", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
