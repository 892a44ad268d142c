"""Fig. 3 (bottom-right) analog on B200:
time to reach a resolution-dependent tolerance tol(N) = tol_1024 (1024/N)^2
("a resolution dependence tolerance, which decreases as N^-2") for
the CJM with the 5-, 9- and 17-point stencils, N = 64 ... 8192 points per
dimension (h = 1/N, N-1 unknowns per side, DESIGN R1), on the test problem of
P:440-453.  Per run: iterations, device time (cjm_solve, inputs resident),
host-to-host time (cjm_solve_host from pinned buffers: the paper's GPU times
include the transfers), GLUPS and the real error vs the analytic solution.

    python scripts/fig3_analog.py [--tol1024 1e-8] [--nmax 8192]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_00103_b200 import cjm, inputs  # noqa: E402


def run(stencil, N, tol, reps=2):
    n = N - 1
    r = 2 if stencil == 17 else 1
    u0, b, h = inputs.test_problem(n, n, r)
    bd = torch.from_numpy(b).cuda()
    bh = torch.from_numpy(b).pin_memory()
    best_dev, best_host = None, None
    for _ in range(reps):
        ud = torch.from_numpy(u0.copy()).cuda()
        with cjm.Plan(stencil, n, n, h, tol) as plan:
            rep = plan.solve(bd, ud, ok=(0, 3, 5))
        if best_dev is None or rep["solve_s"] < best_dev[0]["solve_s"]:
            best_dev = (rep, ud)
        uh = torch.from_numpy(u0.copy()).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with cjm.Plan(stencil, n, n, h, tol) as plan:
            reph = plan.solve_host(bh, uh, ok=(0, 3, 5))
        torch.cuda.synchronize()
        th = time.perf_counter() - t0
        if best_host is None or th < best_host:
            best_host = th
    rep, ud = best_dev
    u = ud.cpu().numpy()[r:r + n, r:r + n]
    err = float(np.max(np.abs(u - inputs.exact_field(n, n, r, h))))
    return dict(stencil=stencil, N=N, tol=tol, status=rep["status"], iterations=rep["iterations"],
                cycles=rep["cycles"], cycle_len=rep["cycle_len"], device_s=rep["solve_s"],
                host_to_host_s=best_host, glups=n * n * rep["iterations"] / rep["solve_s"] / 1e9,
                r_ratio=rep["r_l2"] / rep["r0_l2"], real_error=err, temporal_k=rep["temporal_k"])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--tol1024", type=float, default=1e-8)
    ap.add_argument("--nmax", type=int, default=8192)
    a = ap.parse_args()
    for stencil in (5, 9, 17):
        N = 64
        while N <= a.nmax:
            tol = a.tol1024 * (1024.0 / N) ** 2
            print(json.dumps(run(stencil, N, tol)), flush=True)
            N *= 2
