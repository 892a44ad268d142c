"""One B200 result line per BASELINE.json config: iterations, cycles,
||r||/||r0||, time-to-tol, GLUPS, per-launch HBM fraction, and the bitwise
comparison with the stored oracle digest (tests/golden/oracle_digests.json).

    python scripts/results_table.py [config ...]
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, measured_peaks  # noqa: E402
from paper_1705_00103_b200 import cjm, inputs  # noqa: E402

DIGESTS = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_digests.json")))


def run(name, reps=3):
    st, nx, ny, tol = CONFIGS[name][:4]
    desc = CONFIGS[name][-1]
    r = 2 if st == 17 else 1
    u0, b, h = inputs.test_problem(nx, ny, r)
    bd = torch.from_numpy(b).cuda()
    best = None
    for _ in range(reps):
        ud = torch.from_numpy(u0.copy()).cuda()
        with cjm.Plan(st, nx, ny, h, tol) as plan:
            rep = plan.solve(bd, ud)
        if best is None or rep["solve_s"] < best[0]["solve_s"]:
            best = (rep, ud)
    rep, ud = best
    u = ud.cpu().numpy()[r:r + ny, r:r + nx]
    peak, _ = measured_peaks()
    t_launch = rep["sweep_s"] / max(rep["hot_launches"], 1)
    out = dict(config=name, baseline=desc, stencil=st, n=nx, iterations=rep["iterations"],
               cycles=rep["cycles"], cycle_len=rep["cycle_len"], m_min=rep["m_min"],
               r_ratio=rep["r_l2"] / rep["r0_l2"], time_to_tol_s=rep["solve_s"],
               glups=nx * ny * rep["iterations"] / rep["solve_s"] / 1e9,
               temporal_k=rep["temporal_k"],
               launch_hbm_frac=24.0 * nx * ny / t_launch / 1e9 / peak if rep["hot_launches"] else None)
    d = DIGESTS.get(name)
    if d:
        out["oracle_iterations"] = d["report"]["iterations"]
        out["oracle_bitwise"] = hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest() == d["sha256"]
        idx = np.array(d["sample_index"])
        want = np.array([float.fromhex(v) for v in d["sample_hex"]])
        out["max_rel_diff_sampled"] = float(np.max(np.abs(u.ravel()[idx] - want)) / d["max_abs_u"])
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["cjm9_64", "cjm5_1024", "cjm9_1024", "cjm9_4096", "cjm17_8192"]
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
