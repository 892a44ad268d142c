"""tab:tab01 analog on B200: speed-up factors of
classical Jacobi (j) and the Chebyshev-Jacobi method (cj), serial CPU and GPU,
on the test problem at N = 1024 (1023^2 unknowns, DESIGN R1) for the 5-, 9-
and 17-point stencils, to the same residual tolerance.

GPU times are measured (cjm_solve, METHOD_JACOBI / METHOD_CHEBYSHEV).  The
serial times are the oracle (plain C, ONE thread) timed on a bounded segment
of sweeps and multiplied by the iteration count of the same solve -- a full
serial Jacobi solve at N = 1024 would take hours; the extrapolation is stated
in the output.  The paper's numbers are for a Kepler / Maxwell GPU and an
Opteron / i7 core (context only).

    python scripts/ratio_table.py [--N 1024] [--tol 1e-8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1705_00103_b200 import cjm, inputs  # noqa: E402

PAPER = {5: dict(j_gpu=71, cj=371, cj_gpu=25235), 9: dict(j_gpu=63, cj=441, cj_gpu=21360),
         17: dict(j_gpu=35, cj=361, cj_gpu=12420)}


def gpu_solve(stencil, n, h, tol, u0, b, method):
    bd = torch.from_numpy(b).cuda()
    opts = dict(method=method)
    if method == cjm.METHOD_JACOBI:
        opts.update(jacobi_check=8192, max_cycles=100000)
    best = None
    for _ in range(2):
        ud = torch.from_numpy(u0.copy()).cuda()
        with cjm.Plan(stencil, n, n, h, tol, **opts) as plan:
            rep = plan.solve(bd, ud)
        if best is None or rep["solve_s"] < best["solve_s"]:
            best = rep
    return best


def serial_rate(stencil, u0, b, h, seconds=3.0):
    """oracle sweeps per second on one thread (a bounded segment)."""
    nt = oracle.num_threads()
    oracle.set_num_threads(1)
    try:
        g = oracle.rhs_to_g(stencil, h, b)
        w = [1.0]
        k, t0 = 1, time.perf_counter()
        oracle.sweeps(stencil, u0, g, w, 0, 1)
        per = time.perf_counter() - t0
        k = max(2, int(seconds / max(per, 1e-6)))
        t0 = time.perf_counter()
        oracle.sweeps(stencil, u0, g, w, 0, k)
        return k / (time.perf_counter() - t0), k
    finally:
        oracle.set_num_threads(nt)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--tol", type=float, default=1e-8)
    a = ap.parse_args()
    n = a.N - 1
    out = []
    for stencil in (5, 9, 17):
        r = 2 if stencil == 17 else 1
        u0, b, h = inputs.test_problem(n, n, r)
        cj = gpu_solve(stencil, n, h, a.tol, u0, b, cjm.METHOD_CHEBYSHEV)
        j = gpu_solve(stencil, n, h, a.tol, u0, b, cjm.METHOD_JACOBI)
        rate, k = serial_rate(stencil, u0, b, h)
        t = {"j": j["iterations"] / rate, "j_gpu": j["solve_s"],
             "cj": cj["iterations"] / rate, "cj_gpu": cj["solve_s"]}
        row = dict(stencil=stencil, N=a.N, tol=a.tol,
                   iterations={"j": j["iterations"], "cj": cj["iterations"]},
                   status={"j": j["status"], "cj": cj["status"]},
                   seconds=t, serial="extrapolated: oracle 1 thread, %d sweeps timed" % k,
                   speedup_vs_j={m: t["j"] / t[m] for m in ("j_gpu", "cj", "cj_gpu")},
                   cj_gpu_vs_j_gpu=t["j_gpu"] / t["cj_gpu"], cj_gpu_vs_cj=t["cj"] / t["cj_gpu"],
                   paper_speedup_vs_j=PAPER[stencil])
        print(json.dumps(row), flush=True)
        out.append(row)
