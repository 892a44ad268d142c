"""Write tests/golden/oracle_digests.json: the oracle's full solves at
BASELINE.json's config sizes, stored as (iteration count, report, SHA-256 of
the final interior field, max|u|, and exact values at sampled nodes).

Calls only oracle/ and the seeded input generator; nothing here comes from
the CUDA path.  The GPU parity tests (tests/test_gpu_parity.py) compare the
CUDA solve with these records: same iteration count, sampled values within
1e-10 max|u| (the north_star bar), and the digest for bitwise equality.

Usage: python tests/make_oracle_digests.py [config names ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1705_00103_b200 import inputs  # noqa: E402

OUT = os.environ.get("CJM_DIGESTS_OUT", os.path.join(ROOT, "tests", "golden", "oracle_digests.json"))

# name -> (stencil, nx, ny, tol, init)   (BASELINE.json configs)
CONFIGS = {
    "cjm9_64": (9, 64, 64, 1e-8, "zero"),
    "cjm9_64_rand": (9, 64, 64, 1e-8, "random"),
    "cjm5_1024": (5, 1024, 1024, 1e-8, "zero"),
    "cjm9_1024": (9, 1024, 1024, 1e-8, "zero"),
    "cjm17_1024": (17, 1024, 1024, 1e-8, "zero"),
    "cjm9_4096": (9, 4096, 4096, 1e-8, "zero"),
    "cjm17_8192": (17, 8192, 8192, 1e-8, "zero"),
    "cjm9_16384": (9, 16384, 16384, 1e-8, "zero"),
}

N_SAMPLES = 2048


def sample_index(nx: int, ny: int) -> np.ndarray:
    """Flat interior indices: the four corners, the middle of every edge row
    and column, and N_SAMPLES splitmix64 positions."""
    fixed = [(0, 0), (0, nx - 1), (ny - 1, 0), (ny - 1, nx - 1),
             (0, nx // 2), (ny - 1, nx // 2), (ny // 2, 0), (ny // 2, nx - 1),
             (1, 1), (ny - 2, nx - 2), (ny // 2, nx // 2)]
    idx = [j * nx + i for j, i in fixed]
    z = inputs.splitmix64(12345 + nx * 7 + ny, N_SAMPLES)
    idx += (z % np.uint64(nx * ny)).astype(np.int64).tolist()
    return np.array(idx, dtype=np.int64)


def digest(field: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(field, dtype="<f8").tobytes()).hexdigest()


def run(name: str) -> dict:
    stencil, nx, ny, tol, init = CONFIGS[name]
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init=init)
    t0 = time.time()
    u, rep = oracle.solve(stencil, h, tol, b, u0)
    dt = time.time() - t0
    interior = u[r:r + ny, r:r + nx]
    idx = sample_index(nx, ny)
    flat = interior.ravel()
    return dict(stencil=stencil, nx=nx, ny=ny, h=h, tol=tol, init=init,
                report=rep, sha256=digest(interior),
                max_abs_u=float(np.max(np.abs(interior))),
                sample_index=idx.tolist(),
                sample_hex=[float(v).hex() for v in flat[idx]],
                oracle_seconds=dt, oracle_threads=oracle.num_threads())


def main(names):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for name in names:
        rec = run(name)
        data[name] = rec
        with open(OUT + ".tmp", "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        os.replace(OUT + ".tmp", OUT)
        print(name, rec["report"]["status"], rec["report"]["iterations"],
              f"{rec['oracle_seconds']:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cjm9_64", "cjm9_64_rand", "cjm5_1024", "cjm9_1024", "cjm17_1024"])
