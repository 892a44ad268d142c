"""Pins of the CPU oracle against what the paper and the mathematics fix.

All tests here are CPU-only (-m "not gpu").  None of them re-types the
oracle's own formula: each compares it with an independent route (dense
eigenvalues, the Chebyshev T_P closed form, 50-digit mpmath, dense / sparse
matrices assembled from the golden coefficient table, manufactured-solution
convergence orders, the paper's printed constants).
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import dense
import oracle
from paper_1705_00103_b200 import inputs

STENCILS = (5, 9, 17)


# ----------------------------------------------------------------------------
# Stencil coefficients (Fig. 1, tab:ste2)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("stencil", STENCILS)
def test_golden_table_properties(stencil):
    c = dense.load_stencil(stencil)
    assert len(c) == stencil
    # row-sum zero (annihilates constants) and symmetry
    assert sum(c.values()) == 0
    for (dx, dy), v in c.items():
        assert c[(-dx, -dy)] == v and c[(dy, dx)] == v
    # the printed integer forms: 1/(6h^2)[4 ... 1 ... -20], 1/(72h^2)[64 -4 16 -1 -300]
    if stencil == 9:
        assert [c[(1, 0)] * 6, c[(1, 1)] * 6, c[(0, 0)] * 6] == [4, 1, -20]
    if stencil == 17:
        assert [c[(1, 0)] * 72, c[(2, 0)] * 72, c[(1, 1)] * 72, c[(2, 2)] * 72,
                c[(0, 0)] * 72] == [64, -4, 16, -1, -300]


@pytest.mark.parametrize("stencil", STENCILS)
def test_oracle_coefficients_match_fig1(stencil):
    """Probe the oracle's sweep with unit impulses: with w = 1, u_C = 0, g = 0
    the output at the centre is exactly a_k = -c_k / c_C for the neighbour k
    holding 1.  Compare to the nearest double of the golden rational."""
    coef = dense.load_stencil(stencil)
    r = oracle.reach(stencil)
    n = 2 * r + 1 + 2  # small grid, centre node well inside
    ic = jc = r + 2    # padded index of the probed node
    for (dx, dy), c in coef.items():
        if (dx, dy) == (0, 0):
            continue
        u = np.zeros((n + 2 * r, n + 2 * r))
        u[jc + dy, ic + dx] = 1.0
        g = np.zeros((n, n))
        out = oracle.sweep(stencil, u, g, 1.0)
        want = float(-c / coef[(0, 0)])
        assert out[jc, ic] == want, (dx, dy)
    # D^-1 b scaling: g = (h^2 / c_C) b
    for h in (0.5, 1.0 / 65, 1.0 / 4097):
        want = h * h / float(coef[(0, 0)])
        assert oracle.gscale(stencil, h) == pytest.approx(want, rel=2e-16, abs=0)


# ----------------------------------------------------------------------------
# Spectral bounds (DESIGN R1, R2)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("stencil", STENCILS)
def test_kappa_max_is_paper_constant(stencil):
    km = dense.load_kappa_max()[stencil]
    for n in (4, 16, 1024, 16384):
        _, kmax = oracle.bounds(stencil, n, n)
        assert kmax == float(km)


@pytest.mark.parametrize("stencil", (5, 9))
@pytest.mark.parametrize("nx,ny", [(7, 7), (8, 8), (15, 9), (16, 16), (5, 12)])
def test_kappa_min_equals_dense_eigenvalue(stencil, nx, ny):
    lam = dense.iteration_eigs(stencil, nx, ny)
    kmin, kmax = oracle.bounds(stencil, nx, ny)
    assert abs(kmin - lam[0]) / lam[0] <= 1e-12
    assert lam[-1] < kmax and lam[0] > 0


@pytest.mark.parametrize("nx,ny", [(3, 3), (7, 7), (15, 15), (12, 7)])
def test_kappa17_exact_under_odd_reflection(nx, ny):
    lam = dense.iteration_eigs(17, nx, ny, closure="odd")
    kmin, kmax = oracle.bounds(17, nx, ny)
    assert abs(kmin - lam[0]) / lam[0] <= 1e-12
    assert lam[-1] <= kmax * (1 + 1e-14)


@pytest.mark.parametrize("nx,ny", [(7, 7), (16, 16), (15, 9)])
def test_kappa17_is_lower_bound_with_dirichlet_ghosts(nx, ny):
    """Fixed data in both ghost rings (the test problem's closure): the
    formula is a valid (slightly low) Chebyshev interval end (DESIGN R2)."""
    lam = dense.iteration_eigs(17, nx, ny, closure="dirichlet")
    kmin, kmax = oracle.bounds(17, nx, ny)
    assert kmin <= lam[0] <= kmin * 1.06
    assert lam[-1] < kmax


def test_kappa_wrong_N_convention_is_rejected():
    """Using N = unknowns (instead of unknowns + 1) is 13-30% off: the
    N convention of DESIGN R1 is the one the eigenvalues select."""
    lam = dense.iteration_eigs(9, 8, 8)
    kmin_wrong, _ = oracle.bounds(9, 7, 7)   # formula evaluated at N = 8
    assert abs(kmin_wrong - lam[0]) / lam[0] > 0.1


# ----------------------------------------------------------------------------
# Cycle length and weights
# ----------------------------------------------------------------------------

def _golden_rows(kind):
    rows = []
    with open(os.path.join(dense.GOLDEN, "schedule_examples.txt")) as f:
        for line in f:
            line = line.split("#")[0].split()
            if line and line[0] == kind:
                rows.append(line[1:])
    return rows


def test_spec_worked_example_M6():
    (kmin, kmax, tol, M), = _golden_rows("spec_m")
    assert oracle.m_min(float(kmin), float(kmax), float(tol)) == int(M)


def _m_min_mp(kmin, kmax, tol):
    mpmath.mp.dps = 50
    kmin, kmax = mpmath.mpf(kmin), mpmath.mpf(kmax)
    mu = (kmax + kmin) / (kmax - kmin)
    return int(mpmath.ceil(mpmath.acosh(1 / mpmath.mpf(tol)) / mpmath.acosh(mu)))


@pytest.mark.parametrize("stencil,n", [(9, 64), (5, 1024), (9, 1024), (17, 1024), (9, 4096),
                                       (17, 8192), (9, 16384), (9, 32768), (5, 32768)])
def test_m_min_matches_mpmath(stencil, n):
    kmin, kmax = oracle.bounds(stencil, n, n)
    assert oracle.m_min(kmin, kmax, 1e-8) == _m_min_mp(kmin, kmax, 1e-8)


def test_m_min_is_minimal():
    """1/T_M(mu) <= tol and 1/T_{M-1}(mu) > tol (optimality witness)."""
    mpmath.mp.dps = 50
    for stencil, n, tol in [(9, 64, 1e-8), (5, 256, 1e-6), (17, 100, 1e-10), (9, 31, 1e-3)]:
        kmin, kmax = oracle.bounds(stencil, n, n)
        M = oracle.m_min(kmin, kmax, tol)
        mu = (mpmath.mpf(kmax) + kmin) / (mpmath.mpf(kmax) - kmin)
        T = lambda k: mpmath.cosh(k * mpmath.acosh(mu))
        assert 1 / T(M) <= tol < 1 / T(M - 1)


def test_cycle_len_is_smallest_2a3b():
    smooth = sorted(2 ** a * 3 ** b for a in range(40) for b in range(26) if 2 ** a * 3 ** b < 10 ** 9)
    for m in list(range(1, 400)) + [5092, 6237, 20353, 46997, 81396, 162786, 199371]:
        P, a, b = oracle.cycle_len(m)
        assert P == 2 ** a * 3 ** b
        assert P == next(v for v in smooth if v >= m)


def test_ordering_golden():
    rows = _golden_rows("order")
    assert len(rows) >= 4
    for row in rows:
        a, b, *t = map(int, row)
        assert list(oracle.ordering(a, b)) == t


@pytest.mark.parametrize("a,b", [(0, 0), (1, 0), (0, 1), (3, 2), (2, 4), (6, 4), (8, 4), (0, 8), (14, 1), (10, 4)])
def test_ordering_is_permutation_of_odd(a, b):
    P = 2 ** a * 3 ** b
    t = oracle.ordering(a, b)
    assert sorted(t.tolist()) == list(range(1, 2 * P, 2))


def _cheb_T(P, x):
    """T_P(x) by its closed form (cos / cosh), independent of the weights."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    inside = np.abs(x) <= 1
    out[inside] = np.cos(P * np.arccos(x[inside]))
    xo = x[~inside]
    out[~inside] = np.sign(xo) ** P * np.cosh(P * np.arccosh(np.abs(xo)))
    return out


@pytest.mark.parametrize("stencil,n,tol", [(9, 64, 1e-8), (5, 64, 1e-8), (17, 64, 1e-8),
                                           (9, 16, 1e-6), (9, 100, 1e-10)])
def test_weights_product_identity(stencil, n, tol):
    """prod_k (1 - w_k kappa) = T_P((kmax+kmin-2kappa)/(kmax-kmin)) / T_P(mu):
    the weights are exactly the reciprocals of the mapped Chebyshev zeros."""
    s = oracle.schedule(stencil, n, n, tol)
    kmin, kmax, P, w = s["kappa_min"], s["kappa_max"], s["P"], s["w"]
    assert P <= 1000
    kap = np.concatenate([np.linspace(kmin, kmax, 3001), np.geomspace(kmin, kmax, 1001)])
    prod = np.ones_like(kap)
    for wk in w:
        prod *= 1.0 - wk * kap
    mu = (kmax + kmin) / (kmax - kmin)
    ref = _cheb_T(P, (kmax + kmin - 2 * kap) / (kmax - kmin)) / _cheb_T(P, np.array([mu]))[0]
    bound = 1.0 / _cheb_T(P, np.array([mu]))[0]
    assert np.max(np.abs(prod - ref)) <= 1e-8 * bound
    # damping bound and endpoint equioscillation
    assert np.max(np.abs(prod)) <= tol * (1 + 1e-8)
    assert abs(abs(prod[0]) - bound) <= 1e-8 * bound
    assert abs(abs(prod[3000]) - bound) <= 1e-8 * bound
    # every weight in [1/kmax, 1/kmin]
    assert np.all(w >= 1 / kmax * (1 - 1e-15)) and np.all(w <= 1 / kmin * (1 + 1e-15))


@pytest.mark.parametrize("stencil,n", [(9, 64), (9, 1024), (17, 8192), (9, 16384)])
def test_weights_match_mpmath_zeros(stencil, n):
    """Sorted weights equal 2/[(kmax+kmin) - (kmax-kmin) cos((2m-1) pi / 2P)]
    evaluated at 50 digits (the formula of S:292)."""
    mpmath.mp.dps = 50
    s = oracle.schedule(stencil, n, n, 1e-8)
    kmin, kmax, P, w = mpmath.mpf(s["kappa_min"]), mpmath.mpf(s["kappa_max"]), s["P"], s["w"]
    ws = np.sort(w)
    idx = sorted(set([0, 1, 2, P // 3, P // 2, P - 3, P - 2, P - 1]))
    for i in idx:
        m = P - i   # ascending weights <-> descending zero index
        z = mpmath.cos((2 * m - 1) * mpmath.pi / (2 * P))
        ref = 2 / ((kmax + kmin) - (kmax - kmin) * z)
        assert abs(float((mpmath.mpf(ws[i]) - ref) / ref)) <= 4e-16


@pytest.mark.parametrize("stencil,n", [(9, 64), (9, 1024), (5, 1024), (17, 1024), (9, 4096)])
def test_ordering_suffix_amplification_bounded(stencil, n):
    """Round-off injected at sweep k is multiplied by the suffix product
    prod_{m>k}(1 - w_m kappa); the ordering of DESIGN R3 keeps it <= 1."""
    s = oracle.schedule(stencil, n, n, 1e-8)
    kmin, kmax, w = s["kappa_min"], s["kappa_max"], s["w"]
    kap = np.concatenate([np.linspace(kmin, kmax, 300), np.geomspace(kmin, kmax, 300)])
    logabs = np.log(np.abs(1.0 - np.outer(w, kap)))
    suffix = np.cumsum(logabs[::-1], axis=0)
    assert np.exp(suffix.max()) <= 1.0 + 1e-6


# ----------------------------------------------------------------------------
# Sweep, residual and cycle against dense matrices
# ----------------------------------------------------------------------------

def _rand(shape, seed):
    return inputs.uniform_pm1(seed, int(np.prod(shape))).reshape(shape)


@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("nx,ny", [(8, 8), (7, 9), (12, 5)])
def test_sweep_matches_dense(stencil, nx, ny):
    r = oracle.reach(stencil)
    h = 1.0 / (nx + 1)
    u = _rand((ny + 2 * r, nx + 2 * r), 11 + nx)
    b = _rand((ny, nx), 17 + ny) / (h * h)
    for w in (1.0, 0.37, 123.5):
        got = oracle.sweep(stencil, u, oracle.rhs_to_g(stencil, h, b), w)
        want = dense.dense_sweep(stencil, u, b, h, w)
        assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, w)
        # ghosts untouched
        mask = np.ones_like(u, dtype=bool)
        mask[r:r + ny, r:r + nx] = False
        assert np.array_equal(got[mask], u[mask])
    # w = 0 is the identity
    assert np.array_equal(oracle.sweep(stencil, u, oracle.rhs_to_g(stencil, h, b), 0.0), u)


@pytest.mark.parametrize("stencil", STENCILS)
def test_residual_matches_dense(stencil):
    r = oracle.reach(stencil)
    nx, ny = 9, 8
    h = 1.0 / (nx + 1)
    u = _rand((ny + 2 * r, nx + 2 * r), 5)
    b = _rand((ny, nx), 6) / (h * h)
    res = b - dense.laplacian_h(stencil, u, h)
    l2, li = oracle.residual(stencil, h, b, u)
    assert l2 == pytest.approx(np.linalg.norm(res), rel=1e-13)
    assert li == pytest.approx(np.max(np.abs(res)), rel=1e-13)


@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("n", [8, 12])
def test_cycle_matches_matrix_polynomial(stencil, n):
    """One full cycle = prod_k (I - w_k D^-1 A) applied to the error
    (S:369), with the weights in the oracle's order."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=99)
    ustar = dense.direct_solve(stencil, u0, b, h)
    s = oracle.schedule(stencil, n, n, 1e-8)
    u = u0.copy()
    g = oracle.rhs_to_g(stencil, h, b)
    for wk in s["w"]:
        u = oracle.sweep(stencil, u, g, wk)
    A, _ = dense.operator(stencil, n, n)
    M = A / dense.centre(stencil)
    e = (u0 - ustar)[r:r + n, r:r + n].ravel()
    for wk in s["w"]:
        e = e - wk * (M @ e)
    got = (u - ustar)[r:r + n, r:r + n].ravel()
    assert np.max(np.abs(got - e)) <= 1e-11
    # and the Chebyshev bound holds for the error in the 2-norm
    e0 = (u0 - ustar)[r:r + n, r:r + n].ravel()
    assert np.linalg.norm(got) <= 1e-8 * np.linalg.norm(e0) * 1.01


# ----------------------------------------------------------------------------
# Full solves (P:436-454 test problem)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("stencil", STENCILS)
@pytest.mark.parametrize("init", ["zero", "random"])
def test_solve_one_cycle_chebyshev_bound(stencil, init):
    n = 64
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init=init, seed=inputs.SEED_BASE)
    u, rep = oracle.solve(stencil, h, 1e-8, b, u0)
    assert rep["status"] == "OK" and rep["cycles"] == 1
    assert rep["iterations"] == rep["cycle_len"]
    kmin, kmax = rep["kappa_min"], rep["kappa_max"]
    mu = (kmax + kmin) / (kmax - kmin)
    bound = 1.0 / math.cosh(rep["cycle_len"] * math.acosh(mu))
    assert rep["r_l2"] / rep["r0_l2"] <= bound * (1 + 1e-3)
    # report residuals agree with the dense residual of the returned field
    res = b - dense.laplacian_h(stencil, u, h)
    assert rep["r_l2"] == pytest.approx(np.linalg.norm(res), rel=1e-6)


@pytest.mark.parametrize("stencil,n_direct_err", [(5, 7.69e-7), (9, 1.40e-5), (17, 3.68e-9)])
def test_solve_reaches_direct_solution(stencil, n_direct_err):
    """Converged CJM == the direct sparse solution of the same discrete system;
    its real error is then the discretisation error (63^2 unknowns, h=1/64)."""
    n = 63
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r)
    ustar = dense.direct_solve(stencil, u0, b, h)
    u, rep = oracle.solve(stencil, h, 1e-12, b, u0)
    assert rep["status"] == "OK"
    scale = np.max(np.abs(ustar))
    assert np.max(np.abs(u - ustar)) <= 1e-9 * scale
    ex = inputs.exact_field(n, n, r, h)
    err = np.max(np.abs(u[r:r + n, r:r + n] - ex))
    assert err == pytest.approx(n_direct_err, rel=0.02)


@pytest.mark.parametrize("stencil,order", [(5, 2.0), (9, 2.0), (17, 4.0)])
def test_discretisation_order(stencil, order):
    """Manufactured-solution convergence orders of the stencils (direct solve):
    5-pt 2, 9-pt alpha=2/3 with pointwise RHS 2, 17-pt 4 (DESIGN R7)."""
    r = dense.reach(stencil)
    errs, hs = [], []
    for N in (16, 32, 64, 128):
        n = N - 1
        u0, b, h = inputs.test_problem(n, n, r)
        us = dense.direct_solve(stencil, u0, b, h)
        errs.append(np.max(np.abs(us[r:r + n, r:r + n] - inputs.exact_field(n, n, r, h))))
        hs.append(h)
    slopes = np.diff(np.log(errs)) / np.diff(np.log(hs))
    assert np.all(np.abs(slopes - order) < 0.15), slopes


def test_source_laplacian_matches_finite_differences():
    """The analytic Delta f used by the Mehrstellen RHS vs a fourth-order
    finite-difference Laplacian of f itself (independent of the formula)."""
    d = 1e-3
    x = np.linspace(0.1, 0.9, 9)
    X = np.arange(-2, 3) * d
    for xi in x:
        for yi in x:
            f = inputs.source(xi + X, yi + X)             # 5 x 5 samples around (xi, yi)
            c = np.array([-1, 16, -30, 16, -1]) / (12 * d * d)
            lap = c @ f[2, :] + c @ f[:, 2]
            want = inputs.source_laplacian(np.array([xi]), np.array([yi]))[0, 0]
            assert lap == pytest.approx(want, rel=1e-7, abs=1e-8)


def test_mehrstellen_rhs_makes_the_9_point_fourth_order():
    """9-point alpha=2/3 with b = f + (h^2/12) Delta f (DESIGN R7): order 4
    (SURVEY [V7]: 2.37e-7, 1.48e-8, 9.26e-10, 5.75e-11 at N = 16..128)."""
    errs, hs = [], []
    for N in (16, 32, 64, 128):
        n = N - 1
        u0, b, h = inputs.test_problem(n, n, 1, rhs="mehrstellen")
        us = dense.direct_solve(9, u0, b, h)
        errs.append(np.max(np.abs(us[1:1 + n, 1:1 + n] - inputs.exact_field(n, n, 1, h))))
        hs.append(h)
    slopes = np.diff(np.log(errs)) / np.diff(np.log(hs))
    assert np.all(np.abs(slopes - 4.0) < 0.15), slopes
    assert errs[2] == pytest.approx(9.26e-10, rel=0.03)


def test_fig4_right_17pt_N128_reaches_1e8():
    """the 17-point stencil at N = 128 reaches real error 1e-8."""
    n = 127
    u0, b, h = inputs.test_problem(n, n, 2)
    u, rep = oracle.solve(17, h, 1e-12, b, u0)
    err = np.max(np.abs(u[2:-2, 2:-2] - inputs.exact_field(n, n, 2, h)))
    assert rep["status"] == "OK" and err <= 1e-8


def test_zero_residual_returns_immediately():
    u0 = np.zeros((12, 12))
    b = np.zeros((10, 10))
    u, rep = oracle.solve(9, 1 / 11, 1e-8, b, u0)
    assert rep["status"] == "OK" and rep["iterations"] == 0 and rep["r0_l2"] == 0.0


def test_ascending_order_is_unstable():
    """The ordering matters in fp64 (DESIGN R3): SPEC's ascending order
     blows up at N = 64 where the stable order converges."""
    n = 63
    u0, b, h = inputs.test_problem(n, n, 1)
    s = oracle.schedule(9, n, n, 1e-8)
    u, rep = oracle.solve(9, h, 1e-8, b, u0, weights_override=np.sort(s["w"]))
    assert rep["status"] != "OK"


def test_solve_independent_of_thread_count():
    n = 100
    u0, b, h = inputs.test_problem(n, n, 2, init="random")
    nt = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        u1, r1 = oracle.solve(17, h, 1e-8, b, u0)
        oracle.set_num_threads(max(2, nt))
        u2, r2 = oracle.solve(17, h, 1e-8, b, u0)
    finally:
        oracle.set_num_threads(nt)
    assert np.array_equal(u1, u2) and r1 == r2


def test_invalid_arguments():
    u0, b, h = inputs.test_problem(8, 8, 1)
    for args in [(9, h, 0.0), (9, h, 1.0), (9, -h, 1e-8), (7, h, 1e-8)]:
        _, rep = oracle.solve(args[0], args[1], args[2], b, u0)
        assert rep["status"] == "INVALID"


def test_sweeps_segment_equals_repeated_sweep():
    n = 37
    u0, b, h = inputs.test_problem(n, n + 3, 2, init="random")
    s = oracle.schedule(17, n, n + 3, 1e-8)
    g = oracle.rhs_to_g(17, h, b)
    u = u0
    for k in range(11):
        u = oracle.sweep(17, u, g, s["w"][(s["P"] - 4 + k) % s["P"]])
    assert np.array_equal(oracle.sweeps(17, u0, g, s["w"], s["P"] - 4, 11), u)


# ----------------------------------------------------------------------------
# Power-of-two ordering (order option LEBEDEV2, DESIGN R3)
# ----------------------------------------------------------------------------

def test_cycle_len_pow2_is_smallest_power_of_two():
    for m in list(range(1, 300)) + [5092, 20353, 81396, 199371]:
        P, a = oracle.cycle_len_pow2(m)
        assert P == 2 ** a and P >= m and (P == 1 or P // 2 < m)


def test_lebedev2_theta8_is_the_classical_ordering():
    """For P = 8 the power-of-two recursion gives the Lebedev-Finogenov
    theta_8 = (1, 15, 7, 9, 3, 13, 5, 11) of zero indices 2i-1 (the classical
    stable ordering the generalised 2^a 3^b one reduces to when b = 0)."""
    s = oracle.schedule(9, 6, 6, 0.3, order="lebedev2")
    assert s["P"] >= s["m_min"] and s["b"] == 0
    assert list(oracle.ordering(3, 0)) == [1, 15, 7, 9, 3, 13, 5, 11]


@pytest.mark.parametrize("stencil,n,tol", [(9, 64, 1e-8), (17, 40, 1e-6), (5, 100, 1e-10)])
def test_lebedev2_weights_product_identity_and_stability(stencil, n, tol):
    """The LEBEDEV2 weights are the reciprocals of the mapped zeros of T_P,
    P = 2^a (closed-form T_P identity), and the suffix amplification of the
    order stays <= 1."""
    s = oracle.schedule(stencil, n, n, tol, order="lebedev2")
    kmin, kmax, P, w = s["kappa_min"], s["kappa_max"], s["P"], s["w"]
    assert P == 2 ** s["a"] and P // 2 < s["m_min"] <= P
    assert sorted(s["t"].tolist()) == list(range(1, 2 * P, 2))
    kap = np.concatenate([np.linspace(kmin, kmax, 2001), np.geomspace(kmin, kmax, 501)])
    prod = np.ones_like(kap)
    for wk in w:
        prod *= 1.0 - wk * kap
    mu = (kmax + kmin) / (kmax - kmin)
    ref = _cheb_T(P, (kmax + kmin - 2 * kap) / (kmax - kmin)) / _cheb_T(P, np.array([mu]))[0]
    bound = 1.0 / _cheb_T(P, np.array([mu]))[0]
    assert np.max(np.abs(prod - ref)) <= 1e-8 * bound
    logabs = np.log(np.abs(1.0 - np.outer(w, kap[::5])))
    assert np.exp(np.cumsum(logabs[::-1], axis=0).max()) <= 1.0 + 1e-6


def test_lebedev2_solve_converges_like_lebedev23():
    """A solve with the LEBEDEV2 weights (weights_override) reaches the same
    tolerance in one cycle of its (longer) power-of-two length."""
    n = 63
    u0, b, h = inputs.test_problem(n, n, 1)
    s2 = oracle.schedule(9, n, n, 1e-8, order="lebedev2")
    u, rep = oracle.solve(9, h, 1e-8, b, u0, weights_override=s2["w"])
    assert rep["status"] == "OK" and rep["cycles"] == 1 and rep["iterations"] == s2["P"]
    assert rep["r_l2"] <= 1e-8 * rep["r0_l2"]


# ----------------------------------------------------------------------------
# 17-point odd-reflection closure of the outer ghost ring (DESIGN R12)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("nx,ny", [(7, 7), (9, 6), (12, 11)])
def test_odd_closure_sweep_is_the_odd_extension_operator(nx, ny):
    """With zero boundary data, one oracle sweep under the closure equals
    u + w D^-1 (b - A_odd u) with A_odd assembled from the golden stencil
    table by reflecting every outer-ring neighbour (tests/dense.py,
    closure="odd") -- the operator whose lambda_min the closed form gives."""
    r, h, w = 2, 1.0 / 13, 0.37
    u = np.zeros((ny + 4, nx + 4))
    u[2:-2, 2:-2] = _rand((ny, nx), 5)
    b = _rand((ny, nx), 6)
    got = oracle.sweeps(17, u, oracle.rhs_to_g(17, h, b), np.array([w]), 0, 1, closure="odd")
    A, _ = dense.operator(17, nx, ny, closure="odd")
    ui = u[2:-2, 2:-2].ravel()
    D = dense.centre(17) / (h * h)
    want = ui + w * (b.ravel() - A @ ui / (h * h)) / D
    assert np.max(np.abs(got[2:-2, 2:-2].ravel() - want)) <= 1e-12 * np.max(np.abs(want))


def test_odd_closure_is_exact_for_bilinear_fields():
    """u(mirror) = 2 u_b - u is exact for fields linear across the boundary:
    the reflected outer ring of a + bx + cy + dxy equals the field itself."""
    n = 10
    x = np.arange(-1, n + 3) / (n + 1)
    X, Y = np.meshgrid(x, x)
    f = 0.3 + 1.7 * X - 0.9 * Y + 2.3 * X * Y
    u = f.copy()
    u[[0, -1], :] = 1e30
    u[:, [0, -1]] = 1e30
    got = oracle.odd_closure(u)
    assert np.max(np.abs(got - f)) <= 1e-14


def test_odd_closure_solve_direct_solution_and_fourth_order():
    """Homogeneous problem Delta u = -2 pi^2 sin sin: the closure is exact for
    the odd solution, the solve reaches the direct solution of A_odd, and
    the discretisation error falls at fourth order."""
    errs = []
    for n in (15, 31, 63):
        u0, b, h = inputs.sine_problem(n, 2)
        u, rep = oracle.solve(17, h, 1e-12, b, u0, closure="odd")
        assert rep["status"] == "OK"
        A, _ = dense.operator(17, n, n, closure="odd", sparse=True)
        import scipy.sparse.linalg as spla
        x = spla.spsolve(A.tocsc(), (b * h * h).ravel()).reshape(n, n)
        assert np.max(np.abs(u[2:-2, 2:-2] - x)) <= 1e-9 * np.max(np.abs(x))
        errs.append(np.max(np.abs(u[2:-2, 2:-2] - inputs.sine_exact(n))))
    assert errs[0] / errs[1] > 13 and errs[1] / errs[2] > 13


def test_odd_closure_one_cycle_meets_the_chebyshev_bound():
    """kappa bounds exact for the closure operator: one cycle of P sweeps
    damps the error of a random start by <= tol in the 2-norm (the weights'
    polynomial is bounded by tol on [kappa_min, kappa_max])."""
    n = 24
    u0, b, h = inputs.sine_problem(n, 2, init="random", seed=3)
    s = oracle.schedule(17, n, n, 1e-6)
    A, _ = dense.operator(17, n, n, closure="odd", sparse=True)
    import scipy.sparse.linalg as spla
    x = spla.spsolve(A.tocsc(), (b * h * h).ravel()).reshape(n, n)
    u = oracle.sweeps(17, u0, oracle.rhs_to_g(17, h, b), s["w"], 0, s["P"], closure="odd")
    e0 = np.linalg.norm(u0[2:-2, 2:-2] - x)
    e1 = np.linalg.norm(u[2:-2, 2:-2] - x)
    assert e1 <= 1e-6 * e0 * (1 + 1e-6)
