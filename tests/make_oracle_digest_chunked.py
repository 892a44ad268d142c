"""The oracle's full solve of one digest config, run in resumable chunks
(for a solve longer than one session on the available host): the same steps
as oracle_solve (oracle/cjm_oracle.c) -- r0 from oracle.delta_norms, cycles of
P scheduled sweeps through oracle.sweeps (which double-buffers exactly like
oracle_solve, so any chunking gives the same bits), the stop test of DESIGN
R4 at every cycle boundary -- with the iterate checkpointed after every
chunk.  Calls only oracle/ and the seeded input generator; nothing comes from
the CUDA path.  The record has the fields of tests/make_oracle_digests.py.

    python tests/make_oracle_digest_chunked.py cjm9_16384 --state DIR --budget SECONDS --out FILE

Exit status 0 when the record was written, 3 when the budget ran out first
(run again with the same --state to resume).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from make_oracle_digests import CONFIGS, digest, sample_index  # noqa: E402
from paper_1705_00103_b200 import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--state", required=True)
    ap.add_argument("--budget", type=float, default=3000.0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--max-cycles", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=0, help="max sweeps per chunk (tests)")
    ap.add_argument("--max-chunks", type=int, default=0, help="stop (exit 3) after this many (tests)")
    a = ap.parse_args()
    t_start = time.time()
    stencil, nx, ny, tol, init = CONFIGS[a.name]
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init=init)
    g = oracle.rhs_to_g(stencil, h, b)
    s = oracle.schedule(stencil, nx, ny, tol)
    P, w = s["P"], s["w"]
    sc = abs(oracle.gscale(stencil, h))
    os.makedirs(a.state, exist_ok=True)
    meta_p, u_p = os.path.join(a.state, "meta.json"), os.path.join(a.state, "u.npy")
    if os.path.exists(meta_p):
        meta = json.load(open(meta_p))
        u = np.load(u_p)
        assert meta["name"] == a.name and u.shape == u0.shape
    else:
        s0, m0 = oracle.delta_norms(stencil, u0, g)
        meta = dict(name=a.name, done=0, cycles=0, seconds=0.0, r0_l2=math.sqrt(s0) / sc,
                    r0_linf=m0 / sc, rho_prev=math.sqrt(s0) / sc, status=None)
        u = u0.copy()
    per = None
    chunks = 0
    while meta["status"] is None:
        if a.max_chunks and chunks >= a.max_chunks:
            break
        chunks += 1
        k = meta["done"] % P                    # position in the current cycle
        left = a.budget - (time.time() - t_start)
        count = P - k if per is None else int(min(P - k, max(1, (left - 60.0) / per)))
        if per is None:
            count = min(count, 8)               # calibration chunk
        if a.chunk:
            count = min(count, a.chunk)
        if per is not None and left < 120.0:
            break
        t0 = time.time()
        u = oracle.sweeps(stencil, u, g, w, k, count)
        dt = time.time() - t0
        per = dt / count if per is None else 0.5 * per + 0.5 * dt / count
        meta["done"] += count
        meta["seconds"] += dt
        if meta["done"] % P == 0:               # cycle boundary: the stop test (DESIGN R4)
            meta["cycles"] += 1
            s1, m1 = oracle.delta_norms(stencil, u, g)
            rho = math.sqrt(s1) / sc
            meta["r_l2"], meta["r_linf"] = rho, m1 / sc
            if not math.isfinite(rho):
                meta["status"] = "DIVERGED"
            elif rho <= tol * meta["r0_l2"]:
                meta["status"] = "OK"
            elif rho > 0.5 * meta["rho_prev"]:
                meta["status"] = "STAGNATED"
            elif meta["cycles"] >= a.max_cycles:
                meta["status"] = "NOT_CONVERGED"
            meta["rho_prev"] = rho
        np.save(u_p + ".tmp.npy", u)
        os.replace(u_p + ".tmp.npy", u_p)
        with open(meta_p + ".tmp", "w") as f:
            json.dump(meta, f)
        os.replace(meta_p + ".tmp", meta_p)
        print(f"{a.name}: {meta['done']} / {P * max(1, meta['cycles'] + (meta['status'] is None))} "
              f"sweeps, {meta['seconds']:.0f} s, status {meta['status']}", flush=True)
    if meta["status"] is None:
        sys.exit(3)
    interior = u[r:r + ny, r:r + nx]
    idx = sample_index(nx, ny)
    flat = interior.ravel()
    rec = dict(stencil=stencil, nx=nx, ny=ny, h=h, tol=tol, init=init,
               report=dict(iterations=meta["done"], cycles=meta["cycles"], status=meta["status"],
                           cycle_len=P, m_min=s["m_min"], kappa_min=s["kappa_min"],
                           kappa_max=s["kappa_max"], r0_l2=meta["r0_l2"], r0_linf=meta["r0_linf"],
                           r_l2=meta["r_l2"], r_linf=meta["r_linf"]),
               sha256=digest(interior), max_abs_u=float(np.max(np.abs(interior))),
               sample_index=idx.tolist(), sample_hex=[float(v).hex() for v in flat[idx]],
               oracle_seconds=meta["seconds"], oracle_threads=oracle.num_threads(),
               oracle_run="chunked: oracle.delta_norms + oracle.sweeps, the steps of oracle_solve")
    with open(a.out, "w") as f:
        json.dump({a.name: rec}, f, indent=1, sort_keys=True)
    print(a.name, rec["report"]["status"], rec["report"]["iterations"], rec["sha256"], flush=True)


if __name__ == "__main__":
    main()
