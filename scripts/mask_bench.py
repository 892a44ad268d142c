"""Measurement of the generic-mask path (NEXT-4) on the GPU: per-sweep time
of the mask kernel (cjm_sweeps, CUDA events around the hot launches), GLUPS
and the HBM fraction at its algorithmic 56 B/LUP, plus one
full solve (cjm_plan_mask + cjm_mask_set + cjm_solve) per mask kind.

    python scripts/mask_bench.py [--n 4096] [--count 400] [--solve-n 1024] [--tune]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import measured_peaks  # noqa: E402
from paper_1705_00103_b200 import cjm, inputs, masks  # noqa: E402

BYTES_PER_LUP = 56.0   # u 8 + aW aE aS aN 32 + g 8 read, u' 8 written


def problem(kind, n):
    if kind == "cartesian":
        u0, b, h = inputs.test_problem(n, n, 1)
        return masks.cartesian(n, n, h), u0, b, None
    return (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(n, n)


def dev(mask):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in mask.items()}


def sweeps(kind, n, count, **opts):
    mk, u0, b, _ = problem(kind, n)
    ud, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
    with cjm.MaskPlan(n, n, 1e-6, 2.0 - 1e-6, 1e-8, mask=dev(mk), **opts) as plan:
        plan.sweeps(bd, ud, 0, min(count, 64))                 # warm-up (graphs, clocks)
        rep = plan.sweeps(bd, ud, 0, count)
    t = rep["sweep_s"] / max(rep["hot_launches"], 1)
    peak, src = measured_peaks()
    gbs = BYTES_PER_LUP * n * n / t / 1e9
    return dict(kind=kind, n=n, sweeps=count, **opts, us_per_sweep=1e6 * t, glups=n * n / t / 1e9,
                algo_gbs=gbs, peak_gbs=peak, peak_src=src, frac=gbs / peak,
                launches=rep["kernel_launches"])


def sweeps_n(stencil, n, count):
    """The Cartesian 9- / 17-point stencils as generic (2m+1)^2 masks: the
    kernel streams the present planes + g + u and writes u'."""
    m = 1 if stencil == 9 else 2
    planes = masks.cartesian_n(stencil, n, n, 1.0 / (n + 1))
    u0, b, h = inputs.test_problem(n, n, m)
    ud, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
    dp = [None if c is None else torch.from_numpy(c).cuda() for c in planes]
    present = sum(c is not None for c in planes) - 1
    bpl = 8.0 * (3 + present)
    with cjm.MaskPlanN(n, n, m, 1e-6, 2.0 - 1e-6, 1e-8, planes=dp) as plan:
        plan.sweeps(bd, ud, 0, min(count, 64))
        rep = plan.sweeps(bd, ud, 0, count)
    t = rep["sweep_s"] / max(rep["hot_launches"], 1)
    peak, src = measured_peaks()
    gbs = bpl * n * n / t / 1e9
    return dict(kind=f"cartesian{stencil}_as_{2 * m + 1}x{2 * m + 1}_mask", n=n, sweeps=count,
                bytes_per_lup=bpl, us_per_sweep=1e6 * t, glups=n * n / t / 1e9, algo_gbs=gbs,
                peak_gbs=peak, peak_src=src, frac=gbs / peak)


def solve(kind, n, tol=1e-8):
    mk, u0, b, ex = problem(kind, n)
    kmin, kmax = cjm.cjm_mask_bounds(mk, iters=2000)
    ud, bd = torch.from_numpy(u0.copy()).cuda(), torch.from_numpy(b).cuda()
    with cjm.MaskPlan(n, n, kmin, kmax, tol, mask=dev(mk)) as plan:
        rep = plan.solve(bd, ud, ok=(0, 3, 5))
    out = dict(kind=kind, n=n, tol=tol, kappa_min=kmin, kappa_max=kmax, status=rep["status"],
               iterations=rep["iterations"], cycles=rep["cycles"], cycle_len=rep["cycle_len"],
               r_ratio=rep["r_l2"] / rep["r0_l2"], solve_s=rep["solve_s"],
               glups=n * n * rep["iterations"] / rep["solve_s"] / 1e9)
    if ex is not None:
        out["max_err_vs_exact"] = float(np.max(np.abs(ud.cpu().numpy()[1:-1, 1:-1] - ex)))
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--count", type=int, default=400)
    ap.add_argument("--solve-n", type=int, default=1024)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--square", action="store_true", help="also the (2m+1)^2 generic masks")
    a = ap.parse_args()
    for kind in ("polar", "bipolar", "cartesian"):
        print(json.dumps(sweeps(kind, a.n, a.count)), flush=True)
    if a.square:
        for st in (9, 17):
            print(json.dumps(sweeps_n(st, a.n, a.count)), flush=True)
    if a.tune:
        for cps in (2, 3, 4, 5, 6, 8):
            print(json.dumps(sweeps("polar", a.n, a.count, ctas_per_sm=cps)), flush=True)
    if a.solve_n:
        for kind in ("polar", "bipolar"):
            print(json.dumps(solve(kind, a.solve_n)), flush=True)
