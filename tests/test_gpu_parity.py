"""GPU parity: the CUDA path (called through the C ABI) against the oracle.

Bar (BASELINE.json north_star): the same iteration count, and the final field
within max|du| <= 1e-10 max|u|.  Because kernel and oracle evaluate the same
per-point association (DESIGN R6) with the same weights (bitwise-equal
schedulers, tests/test_abi.py), we additionally expect -- and assert --
bitwise equality of every field.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import ROOT
from paper_1705_00103_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1705_00103_b200 import cjm  # noqa: E402

DIGESTS = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")
REL = 1e-10


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t) -> np.ndarray:
    return t.cpu().numpy()


def oracle_weights(stencil: int, nx: int, ny: int, plan, tol: float = 1e-8) -> np.ndarray:
    """The oracle's own schedule (no oracle input comes from the CUDA path);
    the plan must hold the same weights, bitwise."""
    w = oracle.schedule(stencil, nx, ny, tol)["w"]
    assert np.array_equal(plan.info()["weights"], w)
    return w


def assert_field_parity(got: np.ndarray, want: np.ndarray, r: int):
    gi, wi = got[r:-r, r:-r], want[r:-r, r:-r]
    scale = max(np.max(np.abs(wi)), 1e-300)
    err = np.max(np.abs(gi - wi)) / scale
    assert err <= REL, f"max|du|/max|u| = {err:.3e}"
    assert np.array_equal(gi, wi), f"not bitwise (max rel diff {err:.3e})"
    # ghosts never written
    assert np.array_equal(got[:r], want[:r]) and np.array_equal(got[-r:], want[-r:])
    assert np.array_equal(got[:, :r], want[:, :r]) and np.array_equal(got[:, -r:], want[:, -r:])


# ------------------------------------------------------------ single sweeps
SHAPES = [(8, 8), (64, 64), (100, 37), (257, 300), (513, 70), (1000, 11), (4, 4), (5, 9)]


@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("nx,ny", SHAPES)
@pytest.mark.parametrize("tile_w,variant", [(256, 3), (512, 3), (0, 7)])
def test_one_sweep_bitwise(stencil, nx, ny, tile_w, variant):
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=inputs.SEED_BASE + nx + 7 * ny)
    kw = dict(temporal_k=1) if variant == 7 else {}
    with cjm.Plan(stencil, nx, ny, h, 1e-8, tile_w=tile_w, variant=variant, **kw) as plan:
        w = oracle_weights(stencil, nx, ny, plan)
        g = oracle.rhs_to_g(stencil, h, b)
        for first in (0, 1, plan.P - 1):
            ud = dev(u0)
            plan.sweeps(dev(b), ud, first, 1)
            torch.cuda.synchronize()
            want = oracle.sweep(stencil, u0, g, w[first % plan.P])
            assert_field_parity(host(ud), want, r)


@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("nx,ny,count", [(300, 257, 37), (1030, 515, 20), (64, 64, 324),
                                         (9, 700, 13), (520, 6, 11)])
@pytest.mark.parametrize("temporal_k", (1, 2, 3, 4))
@pytest.mark.parametrize("variant", (3, 7))
def test_sweep_segment_bitwise(stencil, nx, ny, count, temporal_k, variant):
    """A run of sweeps through the CUDA-graph hot loop (spans several graph
    chunks when count > graph_chunk), K sweeps fused per launch (temporal
    blocking), both kernels, vs the oracle sweep by sweep."""
    if stencil == 17 and variant == 7 and temporal_k > 3:
        pytest.skip("the 17-point warp-tiled kernel runs K <= 3 (K = 4: variant 3)")
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=3)
    with cjm.Plan(stencil, nx, ny, h, 1e-8, graph_chunk=4, temporal_k=temporal_k,
                  variant=variant, resident=-1) as plan:
        w = oracle_weights(stencil, nx, ny, plan)
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 5, count)
        g = oracle.rhs_to_g(stencil, h, b)
        u = u0
        for k in range(count):
            u = oracle.sweep(stencil, u, g, w[(5 + k) % plan.P])
        assert_field_parity(host(ud), u, r)


@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("warps,K", [(0, 1), (0, 2), (0, 3), (0, 4), (11, 4), (5, 3), (7, 2)])
@pytest.mark.parametrize("chunk_rows", (1, 7, 64))
@pytest.mark.parametrize("dyn_pct", ("20", "100"))
def test_dynamic_work_items_bitwise(stencil, warps, K, chunk_rows, dyn_pct, monkeypatch):
    """Hot launches whose CTAs take work items of chunk_rows (strip, row)
    units from a device counter (the default last 20% of the units, or all of
    them): same field as the oracle, sweep by sweep."""
    if stencil == 17 and (K > 3 or warps == 11):
        pytest.skip("the 17-point warp-tiled kernel runs K <= 3 with 4, 5 or 7 warps")
    variant = 7
    monkeypatch.setenv("CJM_DYN_PCT", dyn_pct)
    r = oracle.reach(stencil)
    nx, ny, count = 1030, 515, 9
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=17)
    with cjm.Plan(stencil, nx, ny, h, 1e-8, temporal_k=K, variant=variant, chunk_rows=chunk_rows,
                  resident=-1, graph_chunk=2, warps=warps) as plan:
        w = oracle_weights(stencil, nx, ny, plan)
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 2, count)
    g = oracle.rhs_to_g(stencil, h, b)
    u = u0
    for k in range(count):
        u = oracle.sweep(stencil, u, g, w[(2 + k) % len(w)])
    assert_field_parity(host(ud), u, r)


@pytest.mark.parametrize("cfg", [dict(tile_w=256, stages=4, ctas_per_sm=1),
                                 dict(tile_w=512, stages=16, ctas_per_sm=3),
                                 dict(tile_w=256, stages=32, ctas_per_sm=2, graph_chunk=7, variant=3),
                                 dict(tile_w=512, temporal_k=3, stages=6, variant=3),
                                 dict(tile_w=256, temporal_k=4, ctas_per_sm=4, variant=3),
                                 dict(variant=7, temporal_k=1, stages=2),
                                 dict(variant=7, warps=4, temporal_k=4, stages=8, ctas_per_sm=1),
                                 dict(variant=7, temporal_k=3, stages=3),
                                 dict(variant=7, temporal_k=1, stages=8, ctas_per_sm=3),
                                 dict(variant=7, warps=5, temporal_k=4, stages=6),
                                 dict(variant=7, warps=7, temporal_k=2, stages=3),
                                 dict(variant=7, warps=4, temporal_k=3, stages=5, ctas_per_sm=1),
                                 dict(variant=7, temporal_k=4, chunk_rows=24),
                                 dict(variant=7, temporal_k=4, warps=11),
                                 dict(variant=7, temporal_k=4, warps=11, stages=4, chunk_rows=5),
                                 dict(variant=7, temporal_k=3, chunk_rows=-1),
                                 dict(variant=7, temporal_k=2, chunk_rows=100, ctas_per_sm=1)])
def test_launch_configuration_does_not_change_result(cfg):
    nx, ny = 777, 301
    u0, b, h = inputs.test_problem(nx, ny, 1, init="random", seed=5)
    outs = []
    for kw in (dict(), cfg):
        with cjm.Plan(9, nx, ny, h, 1e-8, resident=-1, **kw) as plan:
            ud = dev(u0)
            plan.sweeps(dev(b), ud, 0, 40)
            outs.append(host(ud))
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------ residual
@pytest.mark.parametrize("stencil", (5, 9, 17))
def test_residual_matches_oracle(stencil):  # noqa: D103
    r = oracle.reach(stencil)
    nx, ny = 333, 129
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=8)
    with cjm.Plan(stencil, nx, ny, h, 1e-8) as plan:
        l2, li = plan.residual(dev(b), dev(u0))
    ol2, oli = oracle.residual(stencil, h, b, u0)
    assert l2 == pytest.approx(ol2, rel=1e-12)
    assert li == oli   # max is order-free: bitwise


# ------------------------------------------------------------ full solves
@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("n,init", [(64, "zero"), (64, "random"), (200, "zero"), (129, "random")])
@pytest.mark.parametrize("temporal_k,variant,resident", [(1, 7, -1), (2, 7, -1), (2, 3, -1), (4, 3, -1),
                                                          (3, 0, -1), (0, 0, 1), (3, 7, -1), (4, 0, -1)])
def test_solve_matches_oracle(stencil, n, init, temporal_k, variant, resident):
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init=init)
    uo, ro = oracle.solve(stencil, h, 1e-8, b, u0)
    with cjm.Plan(stencil, n, n, h, 1e-8, temporal_k=temporal_k, variant=variant,
                  resident=resident) as plan:
        assert plan.info()["resident"] == (1 if resident == 1 else 0)
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"] and rep["cycles"] == ro["cycles"]
    assert rep["r0_l2"] == pytest.approx(ro["r0_l2"], rel=1e-12)
    assert rep["r_l2"] == pytest.approx(ro["r_l2"], rel=1e-9)
    assert_field_parity(host(ud), uo, r)


@pytest.mark.parametrize("temporal_k", (1, 3))
def test_solve_nonsquare_ragged(temporal_k):
    nx, ny = 301, 157
    u0, b, h = inputs.test_problem(nx, ny, 2)
    uo, ro = oracle.solve(17, h, 1e-8, b, u0)
    with cjm.Plan(17, nx, ny, h, 1e-8, temporal_k=temporal_k) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["iterations"] == ro["iterations"]
    assert_field_parity(host(ud), uo, 2)


def test_solve_host_equals_solve_device():
    n = 200
    u0, b, h = inputs.test_problem(n, n, 1)
    with cjm.Plan(9, n, n, h, 1e-8) as plan:
        ud = dev(u0)
        rd = plan.solve(dev(b), ud)
        uh = u0.copy()
        rh = plan.solve_host(b, uh)
    assert rd["iterations"] == rh["iterations"]
    assert np.array_equal(host(ud), uh)
    assert rh["h2d_bytes"] == (u0.size + b.size) * 8 and rh["d2h_bytes"] == b.size * 8


def test_zero_residual_returns_immediately():
    u0 = np.zeros((66, 66))
    b = np.zeros((64, 64))
    with cjm.Plan(9, 64, 64, 1 / 65, 1e-8) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and rep["iterations"] == 0 and rep["r0_l2"] == 0.0


def test_ascending_order_fails_like_oracle():
    n = 63
    u0, b, h = inputs.test_problem(n, n, 1)
    s = oracle.schedule(9, n, n, 1e-8)
    _, ro = oracle.solve(9, h, 1e-8, b, u0, weights_override=np.sort(s["w"]))
    with cjm.Plan(9, n, n, h, 1e-8, order=cjm.ORDER_ASCENDING) as plan:
        rep = plan.solve(dev(b), dev(u0), ok=(0, 3, 4, 5))
    assert rep["status"] != "CJM_OK" and ro["status"] != "OK"


def test_jacobi_method_matches_oracle_sweeps():
    """Classical Jacobi (w = 1, the paper's baseline P:298-300) through the same kernel."""
    n = 48
    u0, b, h = inputs.test_problem(n, n, 1)
    with cjm.Plan(5, n, n, h, 1e-3, method=cjm.METHOD_JACOBI, jacobi_check=100, max_cycles=3) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud, ok=(0, 3))
    g = oracle.rhs_to_g(5, h, b)
    u = u0
    for _ in range(rep["iterations"]):
        u = oracle.sweep(5, u, g, 1.0)
    assert rep["iterations"] == 300
    assert_field_parity(host(ud), u, 1)


def test_too_deep_ring_is_invalid_arg():
    with pytest.raises(cjm.CJMError) as e:
        cjm.Plan(9, 4096, 4096, 1 / 4097, 1e-8, stages=32, variant=7, warps=4)
    assert e.value.name == "CJM_ERR_INVALID_ARG"


@pytest.mark.parametrize("kw", [dict(variant=7, warps=6), dict(variant=3, warps=5), dict(warps=-1),
                                dict(variant=7, temporal_k=3, warps=11), dict(variant=4),
                                dict(variant=5), dict(variant=6),
                                dict(variant=8), dict(variant=7, temporal_k=5),
                                dict(variant=7, temporal_k=4, stages=2)])
def test_invalid_launch_options_are_invalid_arg(kw):
    with pytest.raises(cjm.CJMError) as e:
        cjm.Plan(9, 256, 256, 1 / 257, 1e-8, **kw)
    assert e.value.name == "CJM_ERR_INVALID_ARG"


def test_17_point_k4_falls_back_to_the_shared_line_kernel():
    r = 2
    u0, b, h = inputs.test_problem(300, 200, r, init="random", seed=29)
    with pytest.raises(cjm.CJMError):
        cjm.Plan(17, 300, 200, h, 1e-8, temporal_k=4, variant=7)
    with cjm.Plan(17, 300, 200, h, 1e-8, temporal_k=4) as plan:   # default variant: falls back
        assert plan.info()["variant"] == 3 and plan.info()["temporal_k"] == 4
        w = oracle_weights(17, 300, 200, plan)
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 0, 9)
    g = oracle.rhs_to_g(17, h, b)
    want = oracle.sweeps(17, u0, g, w, 0, 9)
    assert_field_parity(host(ud), want, r)


def test_mehrstellen_rhs_solve_is_fourth_order_accurate():
    """9-point solve with the Mehrstellen RHS (DESIGN R7) to tol 1e-12: the
    oracle's field bitwise, and the real error at the direct solve's
    fourth-order level (5.75e-11 at N = 128, SURVEY [V7])."""
    n = 127
    u0, b, h = inputs.test_problem(n, n, 1, rhs="mehrstellen")
    uo, ro = oracle.solve(9, h, 1e-12, b, u0)
    with cjm.Plan(9, n, n, h, 1e-12) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and rep["iterations"] == ro["iterations"]
    assert_field_parity(host(ud), uo, 1)
    err = np.max(np.abs(host(ud)[1:-1, 1:-1] - inputs.exact_field(n, n, 1, h)))
    assert err <= 1e-10


def test_bad_pitch_is_invalid_arg():
    import ctypes as C
    u0, b, h = inputs.test_problem(64, 64, 1)
    with cjm.Plan(9, 64, 64, h, 1e-8) as plan:
        ud, bd = dev(u0), dev(b)
        # pitch 60 < nx + 2r: rejected by the C ABI itself
        st = cjm.lib().cjm_solve(plan._h, C.c_void_p(bd.data_ptr()), 64, C.c_void_p(ud.data_ptr()), 60,
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream), None)
        assert cjm.STATUS[st] == "CJM_ERR_INVALID_ARG"
        st = cjm.lib().cjm_solve(plan._h, None, 64, C.c_void_p(ud.data_ptr()), 66, None, None)
        assert cjm.STATUS[st] == "CJM_ERR_INVALID_ARG"
        with pytest.raises(ValueError):       # shape checked by the binding
            plan.solve(bd, ud[:, :60])


# ------------------------------------------------------------ stored oracle solves
def _digest_cases():
    """(name, temporal_k, resident): every stored case in the default launch
    configuration (the one bench.py times); those up to 8192^2 also with K = 1
    and K = 2 (the 16384^2 target takes ~30 s per solve in the default one)."""
    if not os.path.exists(DIGESTS):
        return []
    with open(DIGESTS) as f:
        recs = json.load(f)
    out = []
    for name in sorted(recs):
        out.append((name, 0, 0))
        if recs[name]["nx"] * recs[name]["ny"] <= 8192 * 8192:
            out += [(name, 1, -1), (name, 2, -1)]
    return out


@pytest.mark.parametrize("name,temporal_k,resident", _digest_cases())
def test_solve_matches_stored_oracle_digest(name, temporal_k, resident):  # noqa: D103
    """Full solves at BASELINE sizes vs the oracle's stored result
    (tests/make_oracle_digests.py): same iterations, sampled nodes within
    1e-10 max|u| and bitwise, and the SHA-256 of the whole interior."""
    with open(DIGESTS) as f:
        rec = json.load(f)[name]
    st, nx, ny, h, tol = rec["stencil"], rec["nx"], rec["ny"], rec["h"], rec["tol"]
    free = torch.cuda.mem_get_info()[0]
    assert free >= 9 * (nx + 4) * (ny + 4) * 8, "a B200 holds every stored case"
    r = oracle.reach(st)
    u0, b, h2 = inputs.test_problem(nx, ny, r, init=rec["init"])
    assert h2 == h
    with cjm.Plan(st, nx, ny, h, tol, temporal_k=temporal_k, resident=resident) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK"
    assert rep["iterations"] == rec["report"]["iterations"]
    u = host(ud)[r:r + ny, r:r + nx]
    flat = u.ravel()
    idx = np.array(rec["sample_index"])
    want = np.array([float.fromhex(v) for v in rec["sample_hex"]])
    err = np.max(np.abs(flat[idx] - want)) / rec["max_abs_u"]
    assert err <= REL
    assert np.array_equal(flat[idx], want)
    assert np.max(np.abs(u)) == rec["max_abs_u"]
    assert hashlib.sha256(np.ascontiguousarray(u, dtype="<f8").tobytes()).hexdigest() == rec["sha256"]


@pytest.mark.parametrize("stencil,n,first", [(9, 16384, 41471), (17, 8192, 20001)])
def test_full_size_segment_bitwise(stencil, n, first):
    """BASELINE full sizes (the 16384^2 target's full solve is also compared
    through its stored digest, test_solve_matches_stored_oracle_digest) in the
    launch configuration bench.py times
    (default plan: K fused sweeps, dynamic work items, boundary fast modes):
    a segment of scheduled sweeps from a random iterate, whole field bitwise
    equal to the oracle's."""
    r = oracle.reach(stencil)
    free = torch.cuda.mem_get_info()[0]
    if free < 8 * (n + 2 * r) * (n + 2 * r) * 8:
        pytest.skip("not enough device memory")
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=23)
    with cjm.Plan(stencil, n, n, h, 1e-8) as plan:
        w = oracle_weights(stencil, n, n, plan)
        count = 2 * plan.info()["temporal_k"] + 1   # two fused launches + a remainder sweep
        ud = dev(u0)
        plan.sweeps(dev(b), ud, first, count)
        got = host(ud)
        del ud
    want = oracle.sweeps(stencil, u0, oracle.rhs_to_g(stencil, h, b), w, first, count)
    assert_field_parity(got, want, r)


# ------------------------------------------------------------ real-error stop (NEXT-3)
@pytest.mark.parametrize("stencil,n,real_tol", [(17, 127, 1e-8), (5, 63, 1e-6), (9, 100, 1e-4)])
def test_real_error_stop_matches_oracle_cycles(stencil, n, real_tol):
    """cjm_solve_ref stops at the first cycle boundary with max|u - u_exact|
    <= real_tol; the oracle, cycle by cycle, must agree on the
    cycle and the field (bitwise)."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r)
    ex = inputs.exact_field(n, n, r, h)
    s = oracle.schedule(stencil, n, n, 1e-8)
    g = oracle.rhs_to_g(stencil, h, b)
    u, cycles = u0, 0
    while True:
        u = oracle.sweeps(stencil, u, g, s["w"], 0, s["P"])
        cycles += 1
        if np.max(np.abs(u[r:-r, r:-r] - ex)) <= real_tol or cycles > 8:
            break
    with cjm.Plan(stencil, n, n, h, 1e-8) as plan:
        ud = dev(u0)
        rep = plan.solve_ref(dev(b), ud, dev(ex), real_tol)
    assert rep["status"] == "CJM_OK" and rep["cycles"] == cycles
    assert rep["iterations"] == cycles * s["P"]
    assert rep["real_error"] == np.max(np.abs(host(ud)[r:-r, r:-r] - ex))
    assert rep["real_error"] <= real_tol
    assert_field_parity(host(ud), u, r)


def test_real_error_below_discretisation_error_does_not_converge():
    n = 63
    u0, b, h = inputs.test_problem(n, n, 1)
    ex = inputs.exact_field(n, n, 1, h)
    with cjm.Plan(9, n, n, h, 1e-8, max_cycles=4) as plan:
        rep = plan.solve_ref(dev(b), dev(u0), dev(ex), 1e-9, ok=(3, 5))
    assert rep["status"] in ("CJM_ERR_STAGNATED", "CJM_ERR_NOT_CONVERGED")
    assert rep["real_error"] > 1e-9


# ------------------------------------------------------------ shared-memory-resident hot path
@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("nx,ny,count", [(64, 64, 324), (300, 257, 37), (130, 1000, 20), (1024, 1024, 16),
                                         (9, 700, 13), (4, 4, 9), (500, 17, 8)])
def test_resident_segment_bitwise(stencil, nx, ny, count):
    """The cooperative shared-memory kernel (one launch for the whole
    segment, neighbour handshakes between CTA slabs) vs the oracle."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=13)
    try:
        plan = cjm.Plan(stencil, nx, ny, h, 1e-8, resident=1)
    except cjm.CJMError as e:
        assert e.name == "CJM_ERR_INVALID_ARG" and nx * ny >= 1024 * 1024
        pytest.skip("grid does not fit in shared memory")
    with plan:
        w = oracle_weights(stencil, nx, ny, plan)
        ud = dev(u0)
        rep = plan.sweeps(dev(b), ud, 3, count)
        assert rep["resident"] == 1 and rep["hot_launches"] == 1
        g = oracle.rhs_to_g(stencil, h, b)
        want = oracle.sweeps(stencil, u0, g, w, 3, count)
        assert_field_parity(host(ud), want, r)


@pytest.mark.parametrize("nx,ny,resident", [(2048, 4, 0), (1200, 4, 1), (1500, 5, 0), (2600, 4, 0)])
def test_resident_17_point_thin_slabs(nx, ny, resident):
    """17-point grids only a few rows high: every resident CTA slab but the
    last must own >= r = 2 rows (it publishes its first / last r rows to its
    neighbours); bitwise vs the oracle."""
    r = 2
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=37)
    with cjm.Plan(17, nx, ny, h, 1e-8, resident=resident) as plan:
        w = oracle_weights(17, nx, ny, plan)
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 1, 24)
    want = oracle.sweeps(17, u0, oracle.rhs_to_g(17, h, b), w, 1, 24)
    assert_field_parity(host(ud), want, r)


# ------------------------------------------------------------ cycles shorter than K (check launch)
@pytest.mark.parametrize("stencil,n,tol", [(9, 4, 0.5), (5, 5, 0.6), (17, 5, 0.7)])
def test_cycle_shorter_than_temporal_k(stencil, n, tol):
    """P < K: the check launch runs one sweep (a configured launch), the rest
    of the cycle the hot path; same iterations and field as the oracle."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=43)
    K = 3 if stencil == 17 else 4
    s = oracle.schedule(stencil, n, n, tol)
    assert s["P"] < K
    uo, ro = oracle.solve(stencil, h, tol, b, u0)
    with cjm.Plan(stencil, n, n, h, tol, temporal_k=K, resident=-1) as plan:
        assert plan.P == s["P"]
        ud = dev(u0)
        rep = plan.solve(dev(b), ud, ok=(0, 3, 5))
    assert rep["status"][len("CJM_"):].replace("ERR_", "") == ro["status"]
    assert rep["iterations"] == ro["iterations"]
    assert_field_parity(host(ud), uo, r)


@pytest.mark.parametrize("check", (2, 3, 5))
def test_jacobi_check_interval_shorter_than_temporal_k(check):
    """Classical Jacobi (w = 1) checked every 2 / 3 / 5 sweeps with K = 4
    fused sweeps per hot launch: the oracle's Jacobi sweeps, bitwise."""
    n, cycles = 300, 4
    u0, b, h = inputs.test_problem(n, n, 1, init="random", seed=47)
    with cjm.Plan(9, n, n, h, 1e-8, method=cjm.METHOD_JACOBI, jacobi_check=check, temporal_k=4,
                  max_cycles=cycles, resident=-1) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud, ok=(3,))
    assert rep["status"] == "CJM_ERR_NOT_CONVERGED" and rep["iterations"] == cycles * check
    want = oracle.sweeps(9, u0, oracle.rhs_to_g(9, h, b), np.ones(check), 0, cycles * check)
    assert_field_parity(host(ud), want, 1)


# ------------------------------------------------------------ power-of-two ordering
@pytest.mark.parametrize("stencil,n", [(9, 200), (17, 129), (5, 300)])
def test_lebedev2_order_solve_matches_oracle(stencil, n):
    """CJM_ORDER_LEBEDEV2 (P = 2^a, classical Lebedev-Finogenov order): the
    plan's weights equal the oracle's power-of-two schedule and the solve
    equals the oracle's solve with those weights, bitwise."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=53)
    s = oracle.schedule(stencil, n, n, 1e-8, order="lebedev2")
    uo, ro = oracle.solve(stencil, h, 1e-8, b, u0, weights_override=s["w"])
    with cjm.Plan(stencil, n, n, h, 1e-8, order=cjm.ORDER_LEBEDEV2) as plan:
        assert plan.P == s["P"] and np.array_equal(plan.info()["weights"], s["w"])
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"]
    assert_field_parity(host(ud), uo, r)


@pytest.mark.gpu
def test_graft_entry_smoke():
    """__graft_entry__.smoke(): 9-pt 64^2 and 17-pt 48^2 solves through the
    C-ABI, bitwise equal to the oracle (the driver's round-end smoke check)."""
    import __graft_entry__
    __graft_entry__.smoke()


# ------------------------------------------------------------ 17-point odd-reflection closure (NEXT-4)
def _interior_parity(got, want, r):
    gi, wi = got[r:-r, r:-r], want[r:-r, r:-r]
    err = np.max(np.abs(gi - wi)) / max(np.max(np.abs(wi)), 1e-300)
    assert err <= REL and np.array_equal(gi, wi), f"max rel diff {err:.3e}"


@pytest.mark.parametrize("nx,ny", [(64, 64), (300, 257), (1030, 515), (5, 9), (513, 70)])
@pytest.mark.parametrize("problem", ("sine", "exp"))
def test_odd_closure_sweeps_bitwise(nx, ny, problem):
    """cjm_options.closure = ODD (DESIGN R12): the outer ghost ring reflected
    from the iterate before every sweep; the oracle's closure sweeps, bitwise
    (interior; the caller's outer ring is never written)."""
    r = 2
    if problem == "sine" and nx == ny:
        u0, b, h = inputs.sine_problem(nx, r, init="random", seed=73)
    else:
        u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=73)
    with cjm.Plan(17, nx, ny, h, 1e-8, closure=cjm.CLOSURE_ODD) as plan:
        info = plan.info()
        assert info["temporal_k"] == 1 and info["resident"] == 0
        w = oracle_weights(17, nx, ny, plan)
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 4, 13)
        l2, li = plan.residual(dev(b), dev(u0))
    g = oracle.rhs_to_g(17, h, b)
    want = oracle.sweeps(17, u0, g, w, 4, 13, closure="odd")
    got = host(ud)
    _interior_parity(got, want, r)
    assert np.array_equal(got[:2], u0[:2]) and np.array_equal(got[:, :2], u0[:, :2])
    ol2, oli = oracle.residual(17, h, b, oracle.odd_closure(u0))
    assert l2 == pytest.approx(ol2, rel=1e-12) and li == oli


@pytest.mark.parametrize("n", (63, 200))
def test_odd_closure_solve_matches_oracle(n):
    """A whole solve under the closure: same iterations and field as the
    oracle's closure solve; on the homogeneous sine problem the closure is
    exact and the 17-point solve is fourth-order accurate."""
    r = 2
    u0, b, h = inputs.sine_problem(n, r)
    uo, ro = oracle.solve(17, h, 1e-10, b, u0, closure="odd")
    with cjm.Plan(17, n, n, h, 1e-10, closure=cjm.CLOSURE_ODD) as plan:
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and ro["status"] == "OK"
    assert rep["iterations"] == ro["iterations"]
    _interior_parity(host(ud), uo, r)
    err = np.max(np.abs(host(ud)[r:-r, r:-r] - inputs.sine_exact(n)))
    assert err <= 6e-7 * (64 / (n + 1)) ** 4


@pytest.mark.parametrize("kw", [dict(temporal_k=2), dict(resident=1), dict(band_split=1)])
def test_odd_closure_options_are_invalid_arg(kw):
    with pytest.raises(cjm.CJMError) as e:
        cjm.Plan(17, 64, 64, 1 / 65, 1e-8, closure=cjm.CLOSURE_ODD, **kw)
    assert e.value.name == "CJM_ERR_INVALID_ARG"
    with pytest.raises(cjm.CJMError):
        cjm.Plan(9, 64, 64, 1 / 65, 1e-8, closure=cjm.CLOSURE_ODD)
