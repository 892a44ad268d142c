"""GPU parity of the generic 5-point mask path (NEXT-4, tab:ste1,
tab:ste2) against the oracle's mask functions (oracle_mask_sweep /
oracle_mask_residual / oracle_mask_solve), through the C ABI
(cjm_plan_mask, cjm_mask_set, cjm_sweeps, cjm_residual, cjm_solve).

Iterates must be bit-identical (same per-node DAG, DESIGN R10); residual
norms agree to 1e-12 relative (different summation order)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1705_00103_b200 import cjm, inputs, masks

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def problem(kind, nx, ny):
    if kind == "cartesian":
        u0, b, h = inputs.test_problem(nx, ny, 1)
        return masks.cartesian(nx, ny, h), u0, b
    mk, u0, b, _ = (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(nx, ny)
    return mk, u0, b


def oracle_weights(kmin, kmax, tol):
    m = oracle.m_min(kmin, kmax, tol)
    P, a, b = oracle.cycle_len(m)
    return m, oracle.weights(kmin, kmax, oracle.ordering(a, b))


def dev(mask):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in mask.items()}


def bounds(mask):
    return cjm.cjm_mask_bounds(mask, iters=3000)


@pytest.mark.parametrize("kind", ["polar", "bipolar", "cartesian"])
def test_mask_plan_schedule_equals_oracle(kind):
    mk, _, _ = problem(kind, 40, 33)
    kmin, kmax = bounds(mk)
    with cjm.MaskPlan(40, 33, kmin, kmax, 1e-8, mask=dev(mk)) as plan:
        info = plan.info()
    m, w = oracle_weights(kmin, kmax, 1e-8)
    assert info["m_min"] == m and info["cycle_len"] == len(w)
    assert np.array_equal(info["weights"], w)


@pytest.mark.parametrize("kind", ["polar", "bipolar", "cartesian"])
@pytest.mark.parametrize("nx,ny", [(4, 4), (37, 21), (300, 77), (520, 260), (256, 300)])
@pytest.mark.parametrize("first,count", [(0, 1), (3, 5)])
def test_mask_sweeps_bitwise(kind, nx, ny, first, count):
    mk, u0, b = problem(kind, nx, ny)
    u = u0.copy()
    u[1:-1, 1:-1] = inputs.uniform_pm1(11 + nx, nx * ny).reshape(ny, nx)
    kmin, kmax = bounds(mk)
    with cjm.MaskPlan(nx, ny, kmin, kmax, 1e-8, mask=dev(mk)) as plan:
        _, w = oracle_weights(kmin, kmax, 1e-8)     # the oracle's own inputs
        assert np.array_equal(plan.info()["weights"], w)
        ud = torch.from_numpy(u.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, first, count)
        got = ud.cpu().numpy()
    want = u.copy()
    for k in range(count):
        want = oracle.mask_sweep(mk, want, b, float(w[(first + k) % len(w)]))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
@pytest.mark.parametrize("nx,ny", [(37, 21), (520, 260)])
def test_mask_residual_matches_oracle(kind, nx, ny):
    mk, u0, b = problem(kind, nx, ny)
    u = u0.copy()
    u[1:-1, 1:-1] = inputs.uniform_pm1(5, nx * ny).reshape(ny, nx)
    kmin, kmax = bounds(mk)
    with cjm.MaskPlan(nx, ny, kmin, kmax, 1e-8, mask=dev(mk)) as plan:
        l2, li = plan.residual(torch.from_numpy(b).cuda(), torch.from_numpy(u).cuda())
    ol2, oli = oracle.mask_residual(mk, u, b)
    assert l2 == pytest.approx(ol2, rel=1e-12)
    assert li == oli


@pytest.mark.parametrize("kind", ["polar", "bipolar", "cartesian"])
@pytest.mark.parametrize("n", [64, 129])
def test_mask_solve_bitwise(kind, n):
    mk, u0, b = problem(kind, n, n - 7)
    kmin, kmax = bounds(mk)
    uo, ro = oracle.mask_solve(mk, b, u0, kmin, kmax, 1e-8)
    with cjm.MaskPlan(n, n - 7, kmin, kmax, 1e-8, mask=dev(mk)) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        rep = plan.solve(torch.from_numpy(b).cuda(), ud, ok=(0, 3, 5))
        got = ud.cpu().numpy()
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"] and rep["cycles"] == ro["cycles"]
    assert rep["r_l2"] <= 1e-8 * rep["r0_l2"]
    assert rep["r0_l2"] == pytest.approx(ro["r0_l2"], rel=1e-12)
    assert rep["r_l2"] == pytest.approx(ro["r_l2"], rel=1e-9)
    assert np.array_equal(got, uo)


def test_mask_solve_converges_to_the_manufactured_solution():
    """Polar 256^2: the CJM solution is within O(h^2) of u = -e^{xy}."""
    n = 256
    mk, u0, b, ex = masks.polar_problem(n, n)
    kmin, kmax = bounds(mk)
    with cjm.MaskPlan(n, n, kmin, kmax, 1e-10, mask=dev(mk)) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        rep = plan.solve(torch.from_numpy(b).cuda(), ud)
    err = np.max(np.abs(ud.cpu().numpy()[1:-1, 1:-1] - ex))
    assert rep["status"] == "CJM_OK"
    assert err < 6e-5, err                 # discretisation error ~3.9e-5 at 256 (O(h^2))


def test_mask_jacobi_method_bitwise():
    """method = JACOBI on a mask plan: w = 1 sweeps."""
    mk, u0, b = problem("bipolar", 70, 50)
    kmin, kmax = bounds(mk)
    with cjm.MaskPlan(70, 50, kmin, kmax, 1e-8, mask=dev(mk), method=cjm.METHOD_JACOBI,
                      jacobi_check=16) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, 0, 9)
        got = ud.cpu().numpy()
    want = u0.copy()
    for _ in range(9):
        want = oracle.mask_sweep(mk, want, b, 1.0)
    assert np.array_equal(got, want)


def test_mask_set_required_and_replaceable():
    mk, u0, b = problem("polar", 48, 40)
    kmin, kmax = bounds(mk)
    bd = torch.from_numpy(b).cuda()
    with cjm.MaskPlan(48, 40, kmin, kmax, 1e-8) as plan:
        with pytest.raises(cjm.CJMError) as e:
            plan.sweeps(bd, torch.from_numpy(u0.copy()).cuda(), 0, 1)
        assert e.value.name == "CJM_ERR_INVALID_ARG"
        plan.mask_set(dev(mk))
        w0 = float(oracle_weights(kmin, kmax, 1e-8)[1][0])
        mk2 = {k: v * 3.0 for k, v in masks.bipolar_problem(48, 40)[0].items()}
        plan.mask_set(dev(mk2))              # a new operator, same plan
        ud = torch.from_numpy(u0.copy()).cuda()
        plan.sweeps(bd, ud, 0, 1)
    assert np.array_equal(ud.cpu().numpy(), oracle.mask_sweep(mk2, u0, b, w0))
    with pytest.raises(cjm.CJMError) as e:   # not a mask plan
        with cjm.Plan(5, 48, 40, 1 / 49, 1e-8) as p5:
            lib = cjm.lib()
            t = dev(mk)
            cjm._check(lib.cjm_mask_set(p5._h, *[cjm.C.c_void_p(t[k].data_ptr()) for k in cjm.MASK_KEYS],
                                        48, None), "cjm_mask_set")
    assert e.value.name == "CJM_ERR_INVALID_ARG"


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
def test_mask_sweeps_bitwise_at_bench_size(kind):
    """The bench workload (4096^2) in the launch configuration bench.py times:
    three scheduled sweeps, full-array comparison with the oracle."""
    n = 4096
    mk, u0, b = problem(kind, n, n)
    u = u0.copy()
    u[1:-1, 1:-1] = inputs.uniform_pm1(3, n * n).reshape(n, n)
    kmin, kmax = 1e-6, 2.0 - 1e-6           # bounds only enter through the weights
    with cjm.MaskPlan(n, n, kmin, kmax, 1e-8, mask=dev(mk)) as plan:
        _, w = oracle_weights(kmin, kmax, 1e-8)
        assert np.array_equal(plan.info()["weights"], w)
        ud = torch.from_numpy(u.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, 7, 3)
        got = ud.cpu().numpy()
    want = u
    for k in range(3):
        want = oracle.mask_sweep(mk, want, b, float(w[(7 + k) % len(w)]))
    assert np.array_equal(got, want)


# ----------------------------------------------- generic (2m+1)^2 masks (m = 1, 2)
def dev_planes(planes):
    return [None if c is None else torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in planes]


def _field(m, nx, ny, seed):
    u = inputs.uniform_pm1(seed, (nx + 2 * m) * (ny + 2 * m)).reshape(ny + 2 * m, nx + 2 * m)
    b = inputs.uniform_pm1(seed + 99, nx * ny).reshape(ny, nx)
    return u, b


KB = (1e-3, 1.9)   # bounds only enter through the weights (oracle_weights)


@pytest.mark.parametrize("m", (1, 2))
@pytest.mark.parametrize("nx,ny", [(4, 4), (37, 21), (300, 77), (257, 300), (520, 9)])
@pytest.mark.parametrize("first,count", [(0, 1), (3, 5)])
def test_maskn_sweeps_bitwise(m, nx, ny, first, count):
    """Variable-coefficient (2m+1)^2 masks, every neighbour present: the
    fields of cjm_sweeps equal the oracle's sweep by sweep (DESIGN R11)."""
    planes = masks.random_n(m, nx, ny, seed=nx + 3 * ny + m)
    u, b = _field(m, nx, ny, 5 + nx)
    _, w = oracle_weights(*KB, 1e-8)
    with cjm.MaskPlanN(nx, ny, m, *KB, 1e-8, planes=dev_planes(planes)) as plan:
        assert np.array_equal(plan.info()["weights"], w)
        ud = torch.from_numpy(u.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, first, count)
        got = ud.cpu().numpy()
    want = u.copy()
    for k in range(count):
        want = oracle.maskn_sweep(planes, want, b, float(w[(first + k) % len(w)]))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("stencil", (9, 17))
def test_maskn_absent_planes_bitwise(stencil):
    """The Cartesian 9- / 17-point Laplacians as masks (absent neighbours are
    neither read nor added)."""
    m = 1 if stencil == 9 else 2
    nx, ny = 301, 157
    u0, b, h = inputs.test_problem(nx, ny, m, init="random", seed=9)
    planes = masks.cartesian_n(stencil, nx, ny, h)
    _, w = oracle_weights(*KB, 1e-8)
    with cjm.MaskPlanN(nx, ny, m, *KB, 1e-8, planes=dev_planes(planes)) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, 1, 4)
        got = ud.cpu().numpy()
        l2, li = plan.residual(torch.from_numpy(b).cuda(), torch.from_numpy(u0).cuda())
    want = u0.copy()
    for k in range(4):
        want = oracle.maskn_sweep(planes, want, b, float(w[(1 + k) % len(w)]))
    assert np.array_equal(got, want)
    ol2, oli = oracle.maskn_residual(planes, u0, b)
    assert l2 == pytest.approx(ol2, rel=1e-12) and li == oli


@pytest.mark.parametrize("stencil", (9, 17))
def test_maskn_cartesian_solve_matches_oracle(stencil):
    """Solve to tol with the Cartesian stencils given as generic masks and the
    closed-form bounds: same iterations, bitwise field as the oracle's."""
    m = 1 if stencil == 9 else 2
    n = 95
    u0, b, h = inputs.test_problem(n, n, m)
    kmin, kmax = oracle.bounds(stencil, n, n)
    planes = masks.cartesian_n(stencil, n, n, h)
    uo, ro = oracle.maskn_solve(planes, b, u0, kmin, kmax, 1e-8)
    with cjm.MaskPlanN(n, n, m, kmin, kmax, 1e-8, planes=dev_planes(planes)) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        rep = plan.solve(torch.from_numpy(b).cuda(), ud)
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"]
    assert rep["r_l2"] == pytest.approx(ro["r_l2"], rel=1e-9)
    assert np.array_equal(ud.cpu().numpy(), uo)


def test_maskn_invalid_arguments():
    with pytest.raises(cjm.CJMError):
        cjm.MaskPlanN(32, 32, 3, *KB, 1e-8)
    planes = masks.cartesian_n(9, 32, 32, 1 / 33)
    planes[4] = None                                   # the centre plane is required
    with cjm.MaskPlanN(32, 32, 1, *KB, 1e-8) as plan:
        with pytest.raises(cjm.CJMError):
            plan.mask_set(dev_planes(planes))
        with pytest.raises(cjm.CJMError):              # mask_set first
            plan.sweeps(torch.zeros(32, 32, dtype=torch.float64, device="cuda"),
                        torch.zeros(34, 34, dtype=torch.float64, device="cuda"), 0, 1)


@pytest.mark.parametrize("m", (1, 2))
def test_maskn_sweeps_bitwise_at_bench_size(m):
    n = 4096
    planes = masks.cartesian_n(9 if m == 1 else 17, n, n, 1 / (n + 1))
    u = inputs.uniform_pm1(3, (n + 2 * m) ** 2).reshape(n + 2 * m, n + 2 * m)
    b = inputs.uniform_pm1(4, n * n).reshape(n, n)
    _, w = oracle_weights(*KB, 1e-8)
    with cjm.MaskPlanN(n, n, m, *KB, 1e-8, planes=dev_planes(planes)) as plan:
        ud = torch.from_numpy(u.copy()).cuda()
        plan.sweeps(torch.from_numpy(b).cuda(), ud, 7, 3)
        got = ud.cpu().numpy()
    want = u
    for k in range(3):
        want = oracle.maskn_sweep(planes, want, b, float(w[(7 + k) % len(w)]))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m", (1, 2))
def test_maskn_variable_coefficient_solve_with_numeric_bounds(m):
    """Symmetric variable-coefficient (2m+1)^2 mask, bounds from
    cjm_mask_bounds_n (widened by 1%), solve to tol: converges, same
    iterations and bitwise field as the oracle with the same bounds."""
    nx, ny = 64, 48
    planes = masks.symmetric_n(m, nx, ny, seed=13)
    kmin, kmax = cjm.cjm_mask_bounds_n(planes, iters=20000)
    kmin, kmax = 0.99 * kmin, 1.01 * kmax
    u0, b = _field(m, nx, ny, 21)
    u0[m:m + ny, m:m + nx] = 0.0
    uo, ro = oracle.maskn_solve(planes, b, u0, kmin, kmax, 1e-8)
    with cjm.MaskPlanN(nx, ny, m, kmin, kmax, 1e-8, planes=dev_planes(planes)) as plan:
        ud = torch.from_numpy(u0.copy()).cuda()
        rep = plan.solve(torch.from_numpy(b).cuda(), ud)
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"]
    assert np.array_equal(ud.cpu().numpy(), uo)
