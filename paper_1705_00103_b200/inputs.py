"""Seeded synthetic inputs shared by the tests, bench.py and smoke().

This module holds none of the method's arithmetic: it only samples the
paper's test problem and a seeded random initial guess.  It imports neither
the CUDA binding nor the oracle, so both sides can take their inputs from it.

Test problem (Eqs. Poisson2D / solPoisson2D):
    Delta u = -(x^2 + y^2) e^{xy} on [0,1]^2,  exact solution u = -e^{xy},
    Dirichlet data from the exact solution.
Grid (DESIGN R1): nx x ny interior unknowns, uniform h; node (i,j) sits at
(x, y) = (i h, j h), 1 <= i <= nx, 1 <= j <= ny.  Square grids use
h = 1/(n+1) (so the boundary nodes i = 0 and i = n+1 lie on x = 0 and x = 1).
Non-square grids use h = 1/(nx+1) and the domain [0,1] x [0,(ny+1)h].
r ghost rings (r = 1: 5/9-point, r = 2: 17-point) carry -e^{xy} evaluated at
their own coordinates (the r = 2 outer ring lies at x or y = -h, 1+h; SPEC
S:89 closure, DESIGN R2).

Initial guess: interior zero (P:444-449 gives none), or, for parity
tests that must exercise every mode, U[-1,1) from splitmix64 with seed
1705_00103 + config index.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 170500103

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """n outputs of the splitmix64 generator started at `seed` (uint64)."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    """n doubles uniform in [-1, 1): top 53 bits of splitmix64."""
    z = splitmix64(seed, n) >> np.uint64(11)
    return z.astype(np.float64) * (2.0 ** -52) - 1.0


def grid_h(nx: int, ny: int) -> float:
    return 1.0 / (nx + 1)


def coords(n: int, r: int, h: float) -> np.ndarray:
    """Coordinates of indices 1-r .. n+r (ghosts included)."""
    return np.arange(1 - r, n + r + 1, dtype=np.float64) * h


def exact(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """u(x, y) = -e^{xy} (Eq. solPoisson2D) on the tensor grid y x x."""
    return -np.exp(np.multiply.outer(y, x))


def source(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """f(x, y) = -(x^2 + y^2) e^{xy} (Eq. Poisson2D)."""
    X = x[None, :]
    Y = y[:, None]
    return -(X * X + Y * Y) * np.exp(np.multiply.outer(y, x))


def source_laplacian(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Delta f for f of `source`: e^{xy} (-4 - 8xy - (x^2 + y^2)^2)."""
    X = x[None, :]
    Y = y[:, None]
    r2 = X * X + Y * Y
    return (-4.0 - 8.0 * X * Y - r2 * r2) * np.exp(np.multiply.outer(y, x))


def test_problem(nx: int, ny: int, r: int, *, h: float | None = None,
                 init: str = "zero", seed: int | None = None, rhs: str = "pointwise"):
    """Returns (u0, b, h).

    u0: (ny + 2r, nx + 2r) float64, ghosts = -e^{xy}, interior = init guess.
    b : (ny, nx) float64, the source sampled at the interior nodes
        (rhs="pointwise"), or with the Mehrstellen correction
        b = f + (h^2/12) Delta f (rhs="mehrstellen"), which makes the compact
        9-point alpha=2/3 stencil fourth order (DESIGN R7; SURVEY [V7]).
    """
    if h is None:
        h = grid_h(nx, ny)
    xg, yg = coords(nx, r, h), coords(ny, r, h)
    u0 = exact(xg, yg)
    if init == "zero":
        u0[r:r + ny, r:r + nx] = 0.0
    elif init == "random":
        s = SEED_BASE if seed is None else seed
        u0[r:r + ny, r:r + nx] = uniform_pm1(s, nx * ny).reshape(ny, nx)
    elif init == "exact":
        pass
    else:
        raise ValueError(init)
    b = source(xg[r:r + nx], yg[r:r + ny])
    if rhs == "mehrstellen":
        b = b + (h * h / 12.0) * source_laplacian(xg[r:r + nx], yg[r:r + ny])
    elif rhs != "pointwise":
        raise ValueError(rhs)
    return np.ascontiguousarray(u0), np.ascontiguousarray(b), h


def exact_field(nx: int, ny: int, r: int, h: float) -> np.ndarray:
    """The analytic solution on the interior nodes, (ny, nx)."""
    return exact(np.arange(1, nx + 1) * h, np.arange(1, ny + 1) * h)


def sine_problem(n: int, r: int, *, init: str = "zero", seed: int | None = None):
    """Returns (u0, b, h) of the homogeneous-Dirichlet problem
    Delta u = -2 pi^2 sin(pi x) sin(pi y) on [0,1]^2, exact u = sin(pi x)
    sin(pi y), on the n x n grid (h = 1/(n+1)): boundary nodes exactly 0, the
    17-point outer ring (r = 2) the exact values (odd about the boundary, so
    the odd-reflection closure of DESIGN R12 is exact for it)."""
    h = grid_h(n, n)
    x = coords(n, r, h)
    s = np.sin(np.pi * x)
    u0 = np.multiply.outer(s, s)
    u0[r - 1, :] = u0[-r, :] = 0.0
    u0[:, r - 1] = u0[:, -r] = 0.0
    if init == "zero":
        u0[r:r + n, r:r + n] = 0.0
    elif init == "random":
        u0[r:r + n, r:r + n] = uniform_pm1(SEED_BASE if seed is None else seed, n * n).reshape(n, n)
    elif init != "exact":
        raise ValueError(init)
    si = s[r:r + n]
    b = -2.0 * np.pi * np.pi * np.multiply.outer(si, si)
    return np.ascontiguousarray(u0), np.ascontiguousarray(b), h


def sine_exact(n: int) -> np.ndarray:
    """sin(pi x) sin(pi y) on the interior nodes of the n x n grid."""
    s = np.sin(np.pi * np.arange(1, n + 1) / (n + 1))
    return np.multiply.outer(s, s)
