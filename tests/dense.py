"""Dense / sparse matrix reference machinery for the oracle pins.

Test-only.  Builds the discrete Laplacian directly from the golden
coefficient table (tests/golden/stencils.txt, transcribed from PAPER.md
Fig. 1 and Eqs. 9-points / 17-points / tab:ste2), independently of the
oracle's hand-written per-point arithmetic.
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_stencil(stencil: int) -> dict[tuple[int, int], Fraction]:
    out = {}
    with open(os.path.join(GOLDEN, "stencils.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            s, dx, dy, c = line.split()
            if int(s) == stencil:
                out[(int(dx), int(dy))] = Fraction(c)
    return out


def load_kappa_max() -> dict[int, Fraction]:
    out = {}
    with open(os.path.join(GOLDEN, "kappa_max.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                s, k = line.split()
                out[int(s)] = Fraction(k)
    return out


def reach(stencil: int) -> int:
    return max(max(abs(dx), abs(dy)) for dx, dy in load_stencil(stencil))


def operator(stencil: int, nx: int, ny: int, closure: str = "dirichlet", sparse: bool = False):
    """h^2 * Delta_h as (A, G): A acts on the nx*ny interior unknowns
    (row-major, index (j-1)*nx + (i-1)), G on the padded field's ghost nodes
    (flattened (ny+2r) x (nx+2r) array; only ghost columns are non-zero).

    closure='dirichlet': ghosts hold given data (G carries them).
    closure='odd': homogeneous Dirichlet on the boundary line i=0 / i=n+1 and
    odd reflection for the outer ring (u(-1) = -u(1)); G is then zero.
    """
    coef = load_stencil(stencil)
    r = reach(stencil)
    W = nx + 2 * r
    rows, cols, vals = [], [], []
    grows, gcols, gvals = [], [], []
    for j in range(1, ny + 1):
        for i in range(1, nx + 1):
            row = (j - 1) * nx + (i - 1)
            for (dx, dy), c in coef.items():
                p, q = i + dx, j + dy
                c = float(c)
                if closure == "odd":
                    sgn = 1.0
                    if p <= 0:
                        if p == 0:
                            continue
                        p, sgn = -p, -sgn
                    elif p >= nx + 1:
                        if p == nx + 1:
                            continue
                        p, sgn = 2 * (nx + 1) - p, -sgn
                    if q <= 0:
                        if q == 0:
                            continue
                        q, sgn = -q, -sgn
                    elif q >= ny + 1:
                        if q == ny + 1:
                            continue
                        q, sgn = 2 * (ny + 1) - q, -sgn
                    rows.append(row); cols.append((q - 1) * nx + (p - 1)); vals.append(sgn * c)
                elif 1 <= p <= nx and 1 <= q <= ny:
                    rows.append(row); cols.append((q - 1) * nx + (p - 1)); vals.append(c)
                else:
                    grows.append(row); gcols.append((q - 1 + r) * W + (p - 1 + r)); gvals.append(c)
    A = sp.csr_matrix((vals, (rows, cols)), shape=(nx * ny, nx * ny))
    G = sp.csr_matrix((gvals, (grows, gcols)), shape=(nx * ny, (ny + 2 * r) * W))
    A.sum_duplicates()
    if sparse:
        return A, G
    return A.toarray(), G.toarray()


def centre(stencil: int) -> float:
    return float(load_stencil(stencil)[(0, 0)])


def laplacian_h(stencil: int, u: np.ndarray, h: float) -> np.ndarray:
    """Delta_h u on the interior (ny, nx) of a padded field u."""
    r = reach(stencil)
    ny, nx = u.shape[0] - 2 * r, u.shape[1] - 2 * r
    A, G = operator(stencil, nx, ny, sparse=True)
    ui = u[r:r + ny, r:r + nx].ravel()
    return ((A @ ui + G @ u.ravel()) / (h * h)).reshape(ny, nx)


def dense_sweep(stencil: int, u: np.ndarray, b: np.ndarray, h: float, w: float) -> np.ndarray:
    """u + w D^-1 (b - A u) with the dense matrices."""
    r = reach(stencil)
    ny, nx = b.shape
    res = b - laplacian_h(stencil, u, h)
    D = centre(stencil) / (h * h)
    out = u.copy()
    out[r:r + ny, r:r + nx] += w * res / D
    return out


def direct_solve(stencil: int, u_ghost: np.ndarray, b: np.ndarray, h: float) -> np.ndarray:
    """Exact discrete solution (sparse LU), ghosts as given; padded field."""
    r = reach(stencil)
    ny, nx = b.shape
    A, G = operator(stencil, nx, ny, sparse=True)
    rhs = b.ravel() * h * h - G @ u_ghost.ravel()
    x = spla.spsolve(A.tocsc(), rhs)
    out = u_ghost.copy()
    out[r:r + ny, r:r + nx] = x.reshape(ny, nx)
    return out


def iteration_eigs(stencil: int, nx: int, ny: int, closure: str = "dirichlet") -> np.ndarray:
    """Eigenvalues of D^-1 A (D = the scalar centre coefficient)."""
    A, _ = operator(stencil, nx, ny, closure=closure)
    M = A / centre(stencil)
    return np.linalg.eigvalsh(0.5 * (M + M.T))
