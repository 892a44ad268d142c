"""Pins of the oracle's generic 5-point mask path (NEXT-4; P:380-418,
tab:ste1, tab:ste2) -- CPU only."""
from __future__ import annotations

import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from paper_1705_00103_b200 import inputs, masks


def assemble(mask):
    """Sparse A (interior) and the ghost coupling of a per-node 5-point mask."""
    ny, nx = mask["C"].shape
    W = nx + 2
    rows, cols, vals, g_rows, g_cols, g_vals = [], [], [], [], [], []
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            rows.append(k); cols.append(k); vals.append(mask["C"][j, i])
            for key, di, dj in (("W", -1, 0), ("E", 1, 0), ("S", 0, -1), ("N", 0, 1)):
                p, q = i + di, j + dj
                if 0 <= p < nx and 0 <= q < ny:
                    rows.append(k); cols.append(q * nx + p); vals.append(mask[key][j, i])
                else:
                    g_rows.append(k); g_cols.append((q + 1) * W + (p + 1)); g_vals.append(mask[key][j, i])
    A = sp.csr_matrix((vals, (rows, cols)), shape=(nx * ny, nx * ny))
    G = sp.csr_matrix((g_vals, (g_rows, g_cols)), shape=(nx * ny, (ny + 2) * W))
    return A, G


def test_polar_golden_spec_example():
    """polar at r = 1, dr = dth = 0.1 -> N/S 100, E 105, W 95, C -400."""
    c = masks.polar_coeffs(np.array(1.0), 0.1, 0.1)
    assert c["N"] == pytest.approx(100.0, rel=1e-14) and c["S"] == pytest.approx(100.0, rel=1e-14)
    assert c["E"] == pytest.approx(105.0, rel=1e-14) and c["W"] == pytest.approx(95.0, rel=1e-14)
    assert c["C"] == pytest.approx(-400.0, rel=1e-14)


def test_mask_row_sums_zero_and_bipolar_degenerate():
    for c in (masks.polar_coeffs(np.linspace(0.5, 3, 7), 0.05, 0.2),
              masks.bipolar_coeffs(np.linspace(0.3, 2, 7), np.linspace(0.2, 1.1, 7), 1.3, 0.1, 0.07)):
        tot = c["W"] + c["E"] + c["S"] + c["N"] + c["C"]
        assert np.max(np.abs(tot)) <= 1e-12 * np.max(np.abs(c["C"]))
    z = masks.bipolar_coeffs(np.array(0.0), np.array(0.0), 1.0, 0.1, 0.1)   # cosh nu = cos mu
    assert all(float(v) == 0.0 for v in z.values())


def test_cartesian_mask_is_the_5_point_stencil():
    n = 20
    h = 1.0 / (n + 1)
    mk = masks.cartesian(n, n, h)
    u0, b, _ = inputs.test_problem(n, n, 1, init="random", seed=2)
    a = oracle.mask_sweep(mk, u0, b, 0.7)
    c = oracle.sweep(5, u0, oracle.rhs_to_g(5, h, b), 0.7)
    assert np.max(np.abs(a - c)) <= 1e-13 * np.max(np.abs(c))


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
def test_mask_sweep_and_residual_match_dense(kind):
    nx, ny = 11, 9
    mk, u0, b, _ = (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(nx, ny)
    u = u0.copy()
    u[1:-1, 1:-1] = inputs.uniform_pm1(7, nx * ny).reshape(ny, nx)
    A, G = assemble(mk)
    Au = A @ u[1:-1, 1:-1].ravel() + G @ u.ravel()
    res = b.ravel() - Au
    D = mk["C"].ravel()
    for w in (1.0, 0.3, 17.0):
        want = u[1:-1, 1:-1].ravel() + w * res / D
        got = oracle.mask_sweep(mk, u, b, w)[1:-1, 1:-1].ravel()
        assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, w) * np.max(np.abs(u))
    l2, li = oracle.mask_residual(mk, u, b)
    assert l2 == pytest.approx(np.linalg.norm(res), rel=1e-12)
    assert li == pytest.approx(np.max(np.abs(res)), rel=1e-12)


def _dense_bounds(mk):
    A, _ = assemble(mk)
    M = (A / mk["C"].ravel()[:, None]).toarray()
    ev = np.linalg.eigvals(M)
    assert np.max(np.abs(ev.imag)) <= 1e-9
    return float(ev.real.min()), float(ev.real.max())


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
def test_mask_solve_reaches_direct_solution(kind):
    """CJM with the mask's (dense) spectral bounds converges to the direct
    sparse solution of the same discrete system."""
    nx, ny = 24, 20
    mk, u0, b, ex = (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(nx, ny)
    kmin, kmax = _dense_bounds(mk)
    assert 0 < kmin < kmax < 2
    A, G = assemble(mk)
    ustar = spla.spsolve(A.tocsc(), b.ravel() - G @ u0.ravel()).reshape(ny, nx)
    u, rep = oracle.mask_solve(mk, b, u0, kmin, kmax, 1e-12)
    assert rep["status"] == "OK"
    assert np.max(np.abs(u[1:-1, 1:-1] - ustar)) <= 1e-9 * np.max(np.abs(ustar))


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
def test_mask_discretisation_is_second_order(kind):
    """Manufactured solution u = -e^{xy} in polar / bipolar
    coordinates: the direct solution of the tab:ste2 mask converges at order 2
    (this pins the mask builders, including reading R9's squared factor)."""
    errs, hs = [], []
    for n in (16, 32, 64, 128):
        mk, u0, b, ex = (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(n, n)
        A, G = assemble(mk)
        us = spla.spsolve(A.tocsc(), b.ravel() - G @ u0.ravel()).reshape(n, n)
        errs.append(np.max(np.abs(us - ex)))
        hs.append(1.0 / (n + 1))
    slopes = np.diff(np.log(errs)) / np.diff(np.log(hs))
    assert np.all(slopes > 1.8) and abs(slopes[-1] - 2.0) < 0.08, slopes


def test_bipolar_printed_single_power_factor_is_not_the_laplacian():
    """Reading R9: with tab:ste2's printed factor (cosh nu - cos mu)/a^2 the
    mask does not approximate Delta u (the manufactured error does not vanish
    under refinement); with the squared metric factor it does (order 2)."""
    errs = []
    for n in (16, 32, 64):
        mk, u0, b, ex = masks.bipolar_problem(n, n)
        nu0, nu1, mu0, mu1 = 0.5, 1.5, math.pi / 4, 3 * math.pi / 4
        mu = mu0 + np.arange(1, n + 1) * (mu1 - mu0) / (n + 1)
        nu = nu0 + np.arange(1, n + 1) * (nu1 - nu0) / (n + 1)
        MU, NU = np.meshgrid(mu, nu)
        scale = 1.0 / (np.cosh(NU) - np.cos(MU))         # squared -> single power
        mk1 = {k: v * scale for k, v in mk.items()}
        A, G = assemble(mk1)
        us = spla.spsolve(A.tocsc(), b.ravel() - G @ u0.ravel()).reshape(n, n)
        errs.append(np.max(np.abs(us - ex)))
    assert min(errs) > 1e-2                               # O(1): not a consistent Laplacian


# ----------------------------------------------- generic (2m+1)^2 masks (m = 1, 2)
def assemble_n(planes):
    """Sparse A (interior) and ghost coupling of a per-node (2m+1)^2 mask."""
    m = oracle.maskn_radius(planes)
    s = 2 * m + 1
    ny, nx = planes[m * s + m].shape
    W = nx + 2 * m
    rows, cols, vals, g_rows, g_cols, g_vals = [], [], [], [], [], []
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            for q, c in enumerate(planes):
                if c is None:
                    continue
                dy, dx = q // s - m, q % s - m
                p, r = i + dx, j + dy
                if 0 <= p < nx and 0 <= r < ny:
                    rows.append(k); cols.append(r * nx + p); vals.append(c[j, i])
                else:
                    g_rows.append(k); g_cols.append((r + m) * W + (p + m)); g_vals.append(c[j, i])
    A = sp.csr_matrix((vals, (rows, cols)), shape=(nx * ny, nx * ny))
    G = sp.csr_matrix((g_vals, (g_rows, g_cols)), shape=(nx * ny, (ny + 2 * m) * W))
    return A, G


def _random_field(m, nx, ny, seed):
    u = inputs.uniform_pm1(seed, (nx + 2 * m) * (ny + 2 * m)).reshape(ny + 2 * m, nx + 2 * m)
    b = inputs.uniform_pm1(seed + 99, nx * ny).reshape(ny, nx)
    return u, b


@pytest.mark.parametrize("m,nx,ny", [(1, 7, 5), (1, 12, 9), (2, 7, 6), (2, 11, 13)])
def test_maskn_sweep_and_residual_match_dense(m, nx, ny):
    """u' = u + w D^-1 (b - A u) and r = b - A u with A assembled from the
    planes (every neighbour with its own per-node factor)."""
    planes = masks.random_n(m, nx, ny, seed=5 + m)
    u, b = _random_field(m, nx, ny, 41)
    A, G = assemble_n(planes)
    inner = u[m:m + ny, m:m + nx].ravel()
    r = b.ravel() - (A @ inner + G @ u.ravel())
    cc = planes[m * (2 * m + 1) + m].ravel()
    w = 0.37
    got = oracle.maskn_sweep(planes, u, b, w)
    want = inner + w * r / cc
    assert np.allclose(got[m:m + ny, m:m + nx].ravel(), want, rtol=1e-13, atol=1e-13)
    assert np.array_equal(got[:m], u[:m]) and np.array_equal(got[:, :m], u[:, :m])
    l2, li = oracle.maskn_residual(planes, u, b)
    assert l2 == pytest.approx(np.linalg.norm(r), rel=1e-12)
    assert li == pytest.approx(np.max(np.abs(r)), rel=1e-12)


@pytest.mark.parametrize("stencil", (9, 17))
def test_maskn_cartesian_is_the_builtin_stencil(stencil):
    """The 9- / 17-point Laplacians as generic masks sweep like the built-in
    stencils (Eq. 9-points, Eq. 17-points), up to the association."""
    m = 1 if stencil == 9 else 2
    n = 23
    u0, b, h = inputs.test_problem(n, n, m, init="random", seed=3)
    planes = masks.cartesian_n(stencil, n, n, h)
    w = 1.3
    got = oracle.maskn_sweep(planes, u0, b, w)
    want = oracle.sweep(stencil, u0, oracle.rhs_to_g(stencil, h, b), w)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("stencil,err", [(9, 1.40e-5), (17, 3.68e-9)])
def test_maskn_cartesian_solve_reaches_the_discretisation_error(stencil, err):
    """CJM with the Cartesian stencils given as generic masks and the closed-
    form bounds: converges and its real error is the direct solve's (SURVEY
    [V7] at N = 64)."""
    m = 1 if stencil == 9 else 2
    n = 63
    u0, b, h = inputs.test_problem(n, n, m)
    kmin, kmax = oracle.bounds(stencil, n, n)
    planes = masks.cartesian_n(stencil, n, n, h)
    u, rep = oracle.maskn_solve(planes, b, u0, kmin, kmax, 1e-12)
    assert rep["status"] == "OK"
    e = np.max(np.abs(u[m:-m, m:-m] - inputs.exact_field(n, n, m, h)))
    assert e == pytest.approx(err, rel=0.05)


@pytest.mark.parametrize("m", (1, 2))
def test_maskn_solve_variable_coefficients_reaches_direct_solution(m):
    """A variable-coefficient mask with dense spectral bounds: the CJM
    converges in one cycle to the sparse direct solution."""
    nx, ny = 13, 11
    planes = masks.random_n(m, nx, ny, seed=2 + m)
    u0, b = _random_field(m, nx, ny, 7)
    u0[m:m + ny, m:m + nx] = 0.0
    A, G = assemble_n(planes)
    cc = planes[m * (2 * m + 1) + m].ravel()
    ev = np.linalg.eigvals((A.toarray().T / cc).T)
    kmin, kmax = float(np.min(ev.real)), float(np.max(ev.real))
    assert kmin > 0
    ustar = spla.spsolve(A.tocsc(), b.ravel() - G @ u0.ravel())
    u, rep = oracle.maskn_solve(planes, b, u0, kmin * (1 - 1e-9), kmax * (1 + 1e-9), 1e-10)
    assert rep["status"] == "OK"
    assert np.max(np.abs(u[m:m + ny, m:m + nx].ravel() - ustar)) <= 1e-8 * np.max(np.abs(ustar))
