"""Per-CTA start / end times of one hot launch (diagnostic build with
CJM_DIAG_TIMES, selected by CJM_LIB)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, make_problem  # noqa: E402
from paper_1705_00103_b200 import cjm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cjm9_4096"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 0
st, nx, ny, tol = CONFIGS[cfg][:4]
u0, b, h = make_problem(st, nx, ny, 0, ny)
ud, bd = torch.from_numpy(u0).cuda(), torch.from_numpy(b).cuda()
L = cjm.lib()
L.cjm_diag_times.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong), C.c_int]
with cjm.Plan(st, nx, ny, h, tol, temporal_k=K) as plan:
    rep = plan.sweeps(bd, ud, 1, 200)
    Kp = rep["temporal_k"]
    plan.sweeps(bd, ud, 1, 2 * Kp)      # check-free: one hot launch after the first
    buf = (C.c_ulonglong * 4096)()
    n = L.cjm_diag_times(plan._h, buf, 2048)
raw = np.array(buf[:2 * n], dtype=np.uint64).reshape(n, 2)
t0 = raw[:, 0].min()
s = (raw[:, 0] - t0).astype(np.float64) / 1e3
dur = (raw[:, 1] & np.uint64((1 << 40) - 1)).astype(np.float64) / 1e3
smid = ((raw[:, 1] >> np.uint64(40)) & np.uint64(0xFFF)).astype(int)
nseg = (raw[:, 1] >> np.uint64(52)).astype(int)
e = s + dur
print(json.dumps(dict(config=cfg, K=Kp, ctas=int(n), warps=rep["warps"], stages=rep["stages"],
                      launch_us=float(e.max()), start_us=[float(s.min()), float(np.median(s)), float(s.max())],
                      end_us=[float(e.min()), float(np.median(e)), float(e.max())],
                      dur_us=[float(dur.min()), float(np.median(dur)), float(dur.max())],
                      busy_frac=float(dur.sum() / (n * e.max())))))
order = np.argsort(dur)
print("slowest CTAs (cta, us, sm, segments):", [(int(i), round(float(dur[i]), 1), int(smid[i]), int(nseg[i])) for i in order[-10:]])
print("fastest CTAs:", [(int(i), round(float(dur[i]), 1), int(smid[i]), int(nseg[i])) for i in order[:10]])
print("mean us by segments:", {int(k): round(float(dur[nseg == k].mean()), 1) for k in np.unique(nseg)})
# co-resident pairs: same SM
bysm = {}
for i in range(n):
    bysm.setdefault(int(smid[i]), []).append(i)
pairs = [v for v in bysm.values() if len(v) == 2]
print("SMs with 2 CTAs:", len(pairs), "with 1:", sum(len(v) == 1 for v in bysm.values()),
      "max per SM:", max(len(v) for v in bysm.values()))
print("CTA->SM sample:", [(i, int(smid[i])) for i in range(0, n, 37)])
# per-SM total busy (sum of co-resident CTA durations) vs max
smmax = np.array([max(dur[v]) for v in bysm.values()])
print("per-SM max duration us: min/median/max", round(float(smmax.min()), 1), round(float(np.median(smmax)), 1), round(float(smmax.max()), 1))
# GPC-ish structure: duration by smid
print("dur by smid (sorted by smid, first CTA):", [round(float(dur[bysm[k][0]]), 0) for k in sorted(bysm)][:148])
