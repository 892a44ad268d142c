"""Dynamic work items must not change the field: sweeps with several
chunk_rows settings vs static ranges, bitwise (9-point; any library build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_00103_b200 import cjm, inputs  # noqa: E402

for nx, ny in ((1030, 515), (777, 301), (4096, 4096)):
    u0, b, h = inputs.test_problem(nx, ny, 1, init="random", seed=11)
    bd = torch.from_numpy(b).cuda()
    outs = {}
    for K in (3, 4):
        for ch in (-1, 24, 64, 128, 256):
            with cjm.Plan(9, nx, ny, h, 1e-8, temporal_k=K, variant=7, chunk_rows=ch, resident=-1) as pl:
                ud = torch.from_numpy(u0.copy()).cuda()
                pl.sweeps(bd, ud, 3, 24)
                outs[(K, ch)] = ud.cpu().numpy()
    ref = outs[(3, -1)]
    bad = [k for k, v in outs.items() if not np.array_equal(v, ref)]
    print(nx, ny, "mismatch:" if bad else "all bitwise equal", bad, flush=True)
