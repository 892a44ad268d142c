"""Generic 5-point masks of the paper's tab:ste2 and their test
problems (inputs of the generic-mask path, NEXT-4).

The paper's code is "totally generic regarding discretization and
coordinates: the choice of coordinates determines the discretization of the
Laplacian operator, and this discretization determines the mask of the
functions".  A mask here is the dict of per-node coefficient
arrays W, E, S, N, C (PDE units, each ny x nx) of tab:ste1's upper table
(f_W, f_E, f_S, f_N, f_C; W/E = the first coordinate -/+, S/N = the second
coordinate -/+).  These builders evaluate tab:ste2's rows at the nodes; the
solver (CUDA path) and the oracle both take the resulting arrays as input.

Uniform meshes in the computational coordinates (tab:ste2 caption: "In all
cases we assume uniform meshes").  Node (i, j), 1 <= i <= nx, 1 <= j <= ny,
sits at (q1_0 + i d1, q2_0 + j d2); one ghost ring (i or j = 0, n+1) holds the
Dirichlet data.  Test problems use the paper's exact solution u = -e^{xy}
 mapped through each coordinate system, so Delta u = -(x^2+y^2) e^{xy}.

Reading R9: tab:ste2 prints the bipolar factor as
(cosh nu - cos mu) / a^2; the bipolar Laplacian's metric factor is its square,
((cosh nu - cos mu) / a)^2.  The factor is common to the five coefficients of
a node, so D^-1 A (and the weights) are the same either way; it only scales
the right-hand side.  The builder uses the squared (correct) metric so that
the manufactured-solution test converges to -e^{xy}.
"""
from __future__ import annotations

import math

import numpy as np


def _exact_xy(x, y):
    return -np.exp(x * y)


# Fig. 1 / Eq. 9-points / Eq. 17-points as (2m+1) x (2m+1) coefficient masks
# (PDE units x h^2): offsets (dx, dy) -> coefficient.
_CART9 = {(0, 0): -20.0 / 6.0, (-1, 0): 4.0 / 6.0, (1, 0): 4.0 / 6.0, (0, -1): 4.0 / 6.0,
          (0, 1): 4.0 / 6.0, (-1, -1): 1.0 / 6.0, (1, -1): 1.0 / 6.0, (-1, 1): 1.0 / 6.0,
          (1, 1): 1.0 / 6.0}
_CART17 = {(0, 0): -300.0 / 72.0}
for _d, _c1, _c2 in ((1, 64.0, 16.0), (2, -4.0, -1.0)):
    for _dx, _dy in ((-_d, 0), (_d, 0), (0, -_d), (0, _d)):
        _CART17[(_dx, _dy)] = _c1 / 72.0
    for _dx, _dy in ((-_d, -_d), (_d, -_d), (-_d, _d), (_d, _d)):
        _CART17[(_dx, _dy)] = _c2 / 72.0


def plane_index(m: int, dx: int, dy: int) -> int:
    """Plane of neighbour (i+dx, j+dy) in a (2m+1)^2 mask (row-major, dy major)."""
    return (dy + m) * (2 * m + 1) + (dx + m)


def cartesian_n(stencil: int, nx: int, ny: int, h: float) -> list:
    """The 9-point (m = 1) or 17-point (m = 2) Cartesian Laplacian (alpha =
    2/3, Eq. 9-points / Eq. 17-points) as a generic mask of per-node planes
    (tab:ste1: the most generic data structure); absent neighbours are None."""
    table, m = {9: (_CART9, 1), 17: (_CART17, 2)}[stencil]
    planes = [None] * (2 * m + 1) ** 2
    for (dx, dy), c in table.items():
        planes[plane_index(m, dx, dy)] = np.full((ny, nx), c / (h * h))
    return planes


def random_n(m: int, nx: int, ny: int, seed: int) -> list:
    """A variable-coefficient (2m+1)^2 mask with every neighbour present:
    neighbour coefficients in [0.1, 1), centre = -(sum of |neighbours|) x 1.25
    (strictly diagonally dominant, so D^-1 A has a positive spectrum)."""
    from . import inputs
    q = (2 * m + 1) ** 2
    planes = []
    for k in range(q):
        planes.append(0.55 + 0.45 * inputs.uniform_pm1(seed + k, nx * ny).reshape(ny, nx))
    qc = plane_index(m, 0, 0)
    planes[qc] = -1.25 * sum(planes[k] for k in range(q) if k != qc)
    return planes


def symmetric_n(m: int, nx: int, ny: int, seed: int) -> list:
    """A variable-coefficient (2m+1)^2 mask whose operator is symmetric: every
    edge (node, node + (dx, dy)) gets one weight in [0.1, 1) used by both of
    its nodes, centre = -1.25 x the node's weight sum (so D^-1 A is similar
    to a symmetric positive definite matrix: real, positive spectrum)."""
    from . import inputs
    s = 2 * m + 1
    planes = [None] * (s * s)
    qc = plane_index(m, 0, 0)
    total = np.zeros((ny, nx))
    k = 0
    for dy in range(-m, m + 1):
        for dx in range(-m, m + 1):
            if (dy, dx) <= (0, 0):
                continue                      # each undirected edge once: (dx, dy) > 0
            wgt = 0.55 + 0.45 * inputs.uniform_pm1(seed + k, (ny + 2 * m) * (nx + 2 * m)) \
                .reshape(ny + 2 * m, nx + 2 * m)
            k += 1
            # edge weight stored at the lower endpoint (i, j) of (i, j) -- (i+dx, j+dy)
            fwd = wgt[m:m + ny, m:m + nx]
            bwd = wgt[m - dy:m - dy + ny, m - dx:m - dx + nx]
            planes[plane_index(m, dx, dy)] = fwd.copy()
            planes[plane_index(m, -dx, -dy)] = bwd.copy()
            total += fwd + bwd
    planes[qc] = -1.25 * total
    return planes


def cartesian(nx: int, ny: int, h: float) -> dict:
    """tab:ste2 'Cartesian coordinates' with Dx = Dy = h (the 5-point stencil)."""
    one = np.full((ny, nx), 1.0 / (h * h))
    return dict(W=one.copy(), E=one.copy(), S=one.copy(), N=one.copy(),
                C=np.full((ny, nx), -2.0 / (h * h) - 2.0 / (h * h)))


def polar_coeffs(r: np.ndarray, dr: float, dth: float) -> dict:
    """tab:ste2 'Polar coordinates' at radii r (broadcast over theta):
    W = 1/dr^2 - 1/(2 r dr), E = 1/dr^2 + 1/(2 r dr), S = N = 1/(r^2 dth^2),
    C = -2/dr^2 - 2/(r^2 dth^2)."""
    r = np.asarray(r, dtype=np.float64)
    return dict(W=1.0 / (dr * dr) - 1.0 / (2.0 * r * dr), E=1.0 / (dr * dr) + 1.0 / (2.0 * r * dr),
                S=1.0 / (r * r * dth * dth), N=1.0 / (r * r * dth * dth),
                C=-2.0 / (dr * dr) - 2.0 / (r * r * dth * dth))


def polar_problem(nx: int, ny: int, r0: float = 1.0, r1: float = 2.0, th0: float = 0.0,
                  th1: float = math.pi / 2):
    """Annular sector r in [r0, r1], theta in [th0, th1]; nx radial, ny angular
    unknowns.  Returns (mask, u0 with ghosts, b, exact interior)."""
    dr, dth = (r1 - r0) / (nx + 1), (th1 - th0) / (ny + 1)
    r = r0 + np.arange(0, nx + 2) * dr
    th = th0 + np.arange(0, ny + 2) * dth
    R, TH = np.meshgrid(r, th)                 # (ny+2, nx+2), row = theta
    X, Y = R * np.cos(TH), R * np.sin(TH)
    ex = _exact_xy(X, Y)
    u0 = ex.copy()
    u0[1:-1, 1:-1] = 0.0
    b = (-(X * X + Y * Y) * np.exp(X * Y))[1:-1, 1:-1]
    cf = polar_coeffs(R[1:-1, 1:-1], dr, dth)
    mask = {k: np.ascontiguousarray(np.broadcast_to(v, (ny, nx)), dtype=np.float64) for k, v in cf.items()}
    return mask, np.ascontiguousarray(u0), np.ascontiguousarray(b), np.ascontiguousarray(ex[1:-1, 1:-1])


def bipolar_coeffs(mu: np.ndarray, nu: np.ndarray, a: float, dmu: float, dnu: float) -> dict:
    """tab:ste2 'Bipolar coordinates' (metric factor squared, reading R9):
    F = ((cosh nu - cos mu) / a)^2, W = E = F/dmu^2, S = N = F/dnu^2,
    C = -2F/dmu^2 - 2F/dnu^2."""
    F = ((np.cosh(nu) - np.cos(mu)) / a) ** 2
    return dict(W=F / (dmu * dmu), E=F / (dmu * dmu), S=F / (dnu * dnu), N=F / (dnu * dnu),
                C=-2.0 * F / (dmu * dmu) - 2.0 * F / (dnu * dnu))


def bipolar_problem(nx: int, ny: int, a: float = 1.0, mu0: float = math.pi / 4,
                    mu1: float = 3 * math.pi / 4, nu0: float = 0.5, nu1: float = 1.5):
    """Bipolar patch mu in [mu0, mu1] (along i), nu in [nu0, nu1] (along j)."""
    dmu, dnu = (mu1 - mu0) / (nx + 1), (nu1 - nu0) / (ny + 1)
    mu = mu0 + np.arange(0, nx + 2) * dmu
    nu = nu0 + np.arange(0, ny + 2) * dnu
    MU, NU = np.meshgrid(mu, nu)
    den = np.cosh(NU) - np.cos(MU)
    X, Y = a * np.sinh(NU) / den, a * np.sin(MU) / den
    ex = _exact_xy(X, Y)
    u0 = ex.copy()
    u0[1:-1, 1:-1] = 0.0
    b = (-(X * X + Y * Y) * np.exp(X * Y))[1:-1, 1:-1]
    cf = bipolar_coeffs(MU[1:-1, 1:-1], NU[1:-1, 1:-1], a, dmu, dnu)
    mask = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in cf.items()}
    return mask, np.ascontiguousarray(u0), np.ascontiguousarray(b), np.ascontiguousarray(ex[1:-1, 1:-1])
