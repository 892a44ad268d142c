"""Run a fixed number of scheduled sweeps of one config (for ncu and tuning).

    python scripts/sweep_runner.py --config cjm9_4096 --count 30 [--tile-w 256 --stages 8 --ctas-per-sm 2]
    python scripts/sweep_runner.py --tune        # sweep the launch-configuration grid
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIGS, make_problem  # noqa: E402
from paper_1705_00103_b200 import cjm  # noqa: E402


def run(config, count, warm, digest=False, **kw):
    st, nx, ny, tol = CONFIGS[config][:4]
    u0, b, h = make_problem(st, nx, ny, 0, ny)
    ud, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
    with cjm.Plan(st, nx, ny, h, tol, **kw) as plan:
        if warm:
            plan.sweeps(bd, ud, 1, warm)
        rep = plan.sweeps(bd, ud, 1, count)
        sha = None
        if digest:   # field after warm + count sweeps (bitwise A/B of builds / launch shapes)
            import hashlib
            sha = hashlib.sha256(ud.cpu().numpy().tobytes()).hexdigest()[:16]
    us = 1e6 * rep["sweep_s"] / count
    K = rep["temporal_k"]
    kw = dict(kw, variant=rep["variant"], warps=rep["warps"], stages=rep["stages"], ctas=rep["ctas"],
              temporal_k=K)
    out = dict(config=config, **kw, us_per_sweep=us, glups=nx * ny / (us * 1e-6) / 1e9,
               gbs_per_launch=24.0 * nx * ny / (K * us * 1e-6) / 1e9, lib=os.environ.get("CJM_LIB", ""))
    if digest:
        out["sha"] = sha
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cjm9_4096")
    ap.add_argument("--count", type=int, default=30)
    ap.add_argument("--warm", type=int, default=0)
    ap.add_argument("--tile-w", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--digest", action="store_true")
    ap.add_argument("--temporal-k", type=int, default=0)
    ap.add_argument("--ks", type=lambda v: [int(x) for x in v.split(",")], default=[1, 2, 3, 4])
    ap.add_argument("--variants", type=lambda v: [int(x) for x in v.split(",")], default=[3, 7])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--chunk-rows", type=int, default=0)
    ap.add_argument("--resident", type=int, default=-1)
    ap.add_argument("--stages-list", type=lambda v: [int(x) for x in v.split(",")], default=[4, 8, 12])
    ap.add_argument("--cps-list", type=lambda v: [int(x) for x in v.split(",")], default=[1, 2, 3, 4])
    a = ap.parse_args()
    if a.tune:
        for cfgname in a.config.split(","):
            grid = []
            for var in a.variants:
                tws = (256, 512) if var == 3 else (256,)
                grid += [(var, K, tw, stg, cps) for K in a.ks for tw in tws for stg in a.stages_list
                         for cps in a.cps_list]
            for var, K, tw, stg, cps in grid:
                try:
                    print(json.dumps(run(cfgname, 2400, 240, variant=var, tile_w=tw, stages=stg,
                                         ctas_per_sm=cps, temporal_k=K)), flush=True)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps(dict(config=cfgname, variant=var, tile_w=tw, stages=stg,
                                          ctas_per_sm=cps, temporal_k=K, error=str(e))), flush=True)
    else:
        print(json.dumps(run(a.config, a.count, a.warm, digest=a.digest, tile_w=a.tile_w, stages=a.stages,
                             ctas_per_sm=a.ctas_per_sm, temporal_k=a.temporal_k, variant=a.variant,
                             warps=a.warps, chunk_rows=a.chunk_rows, resident=a.resident)))
