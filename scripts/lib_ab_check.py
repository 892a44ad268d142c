"""Bitwise A/B of two library builds (CJM_LIB selects the build): writes or
compares the fields of scheduled 9-point sweeps for several shapes, K,
warps and work-item settings.  Run once with --save (reference build), then
with --check (candidate build)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1705_00103_b200 import cjm, inputs  # noqa: E402

OUT = "/tmp/lib_ab"
mode = sys.argv[1]
os.makedirs(OUT, exist_ok=True)
bad = 0
for nx, ny in ((300, 257), (1030, 515), (9, 700), (520, 6), (4096, 4096)):
    u0, b, h = inputs.test_problem(nx, ny, 1, init="random", seed=nx + ny)
    bd = torch.from_numpy(b).cuda()
    for K in (1, 2, 3, 4):
        for kw in (dict(), dict(chunk_rows=7), dict(warps=5), dict(warps=11 if K == 4 else 7)):
            with cjm.Plan(9, nx, ny, h, 1e-8, temporal_k=K, variant=7, resident=-1, **kw) as pl:
                ud = torch.from_numpy(u0.copy()).cuda()
                pl.sweeps(bd, ud, 5, 2 * K + 3)
                got = ud.cpu().numpy()
            f = os.path.join(OUT, f"{nx}_{ny}_{K}_{'_'.join(f'{k}{v}' for k, v in kw.items())}.npy")
            if mode == "--save":
                np.save(f, got)
            else:
                ok = np.array_equal(np.load(f), got)
                bad += not ok
                if not ok:
                    print("MISMATCH", f, flush=True)
print("checked" if mode != "--save" else "saved", "mismatches:", bad)
