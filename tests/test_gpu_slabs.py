"""Row-slab decomposition of the CUDA path on ONE GPU (no NCCL).

Each slab is its own plan (world_size=G, external_halo=1: global schedule,
slab geometry, no communicator); the test moves the halo rows between the
slab tensors with device copies laid out by cjm_halo_plan (the same host logic
the NCCL exchange uses) and calls cjm_sweeps one sweep at a time.  Nothing
waits on anything across slabs (all stream-ordered), so this is a legitimate
single-GPU check of the slab kernels and the halo geometry: the gathered field
must be bitwise equal to the single-domain CUDA run and to the oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1705_00103_b200 import inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1705_00103_b200 import cjm  # noqa: E402


@pytest.mark.parametrize("world,stencil,nx,ny", [(2, 9, 300, 257), (4, 17, 130, 97), (3, 5, 64, 200),
                                                 (8, 9, 513, 64)])
@pytest.mark.parametrize("band_split", (0, 1))
def test_slabs_bitwise_equal_single_domain(world, stencil, nx, ny, band_split):
    """band_split=1 runs each sweep as the multi-GPU overlap schedule does:
    boundary-row bands first, then the interior band (which advances n)."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=21)
    nsweeps = 9
    plans, us, bs, msgs = [], [], [], []
    for g in range(world):
        y0, nyl = cjm.cjm_slab(ny, world, g)
        plans.append(cjm.Plan(stencil, nx, ny, h, 1e-8, world_size=world, rank=g, external_halo=1,
                              band_split=band_split, temporal_k=1))
        assert (plans[-1].y0, plans[-1].ny_local) == (y0, nyl)
        us.append(torch.from_numpy(u0[y0:y0 + nyl + 2 * r].copy()).cuda())
        bs.append(torch.from_numpy(b[y0:y0 + nyl].copy()).cuda())
        msgs.append(cjm.cjm_halo_plan(ny, r, world, g))
    for k in range(nsweeps):
        for g in range(world):
            rep = plans[g].sweeps(bs[g], us[g], k, 1)
            if band_split and plans[g].ny_local > 4 * r:
                assert rep["kernel_launches"] >= 5     # 3 band launches + setup
            else:
                assert rep["kernel_launches"] >= 3
        staged = []
        for g in range(world):                       # read every send block first
            for m in msgs[g]:
                staged.append((m["peer"], g, us[g][m["send_row"]:m["send_row"] + m["rows"]].clone()))
        for peer, src, blk in staged:
            m = [x for x in msgs[peer] if x["peer"] == src][0]
            us[peer][m["recv_row"]:m["recv_row"] + m["rows"]] = blk
    field = torch.cat([us[g][r:-r] for g in range(world)]).cpu().numpy()
    with cjm.Plan(stencil, nx, ny, h, 1e-8, temporal_k=1) as whole:
        ud = torch.from_numpy(u0.copy()).cuda()
        whole.sweeps(torch.from_numpy(b).cuda(), ud, 0, nsweeps)
        ref = ud.cpu().numpy()
    s = oracle.schedule(stencil, nx, ny, 1e-8)
    uo = oracle.sweeps(stencil, u0, oracle.rhs_to_g(stencil, h, b), s["w"], 0, nsweeps)
    assert np.array_equal(field, ref[r:-r])
    assert np.array_equal(field, uo[r:-r])
    # slab-local residuals combine to the global one
    l2s, lis = zip(*[plans[g].residual(bs[g], us[g]) for g in range(world)])
    gl2, gli = oracle.residual(stencil, h, b, np.concatenate([u0[:r], field, u0[-r:]]))
    assert np.sqrt(sum(x * x for x in l2s)) == pytest.approx(gl2, rel=1e-12)
    assert max(lis) == gli
    for p in plans:
        p.close()


@pytest.mark.parametrize("world,stencil,nx,ny", [(2, 9, 300, 257), (4, 17, 130, 97), (3, 5, 200, 64),
                                                 (8, 9, 513, 200)])
@pytest.mark.parametrize("K,variant", [(2, 0), (3, 3), (2, 3), (4, 0), (3, 7), (2, 77), (4, 77)])
@pytest.mark.parametrize("band_split", (0, 1))
def test_deep_halo_slabs_bitwise(world, stencil, nx, ny, K, variant, band_split):
    """K sweeps fused per launch across slabs: H = K r deep halos (u with H
    ghost rows, rhs with H extra rows, refreshed after every launch), the
    ghost rows inside the global grid computed redundantly, bitwise equal to
    the whole-domain oracle."""
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=31)
    nsweeps = 12
    plans = []
    for g in range(world):
        kw = dict(world_size=world, rank=g, external_halo=1, temporal_k=K, band_split=band_split)
        if variant == 77:      # variant 7 with small dynamic work items (band launches too)
            kw.update(variant=7, chunk_rows=5)
        elif variant:
            kw["variant"] = variant
        if stencil == 17 and variant in (7, 77) and K > 3:
            kw["variant"] = 3
        plans.append(cjm.Plan(stencil, nx, ny, h, 1e-8, **kw))
    H = plans[0].ghost_rows
    if plans[0].info()["temporal_k"] != K:
        pytest.skip("slabs too thin for this K (plan fell back to K=1)")
    assert H == K * r and plans[0].rhs_ghost_rows == H
    u_pad = np.pad(u0, ((H - r, H - r), (0, 0)))
    b_pad = np.pad(b, ((H, H), (0, 0)))
    us, bs, msgs = [], [], []
    for g in range(world):
        y0, nyl = cjm.cjm_slab(ny, world, g)
        us.append(torch.from_numpy(u_pad[y0:y0 + nyl + 2 * H].copy()).cuda())
        bs.append(torch.from_numpy(b_pad[y0:y0 + nyl + 2 * H].copy()).cuda())
        msgs.append(cjm.cjm_halo_plan(ny, H, world, g))
    for k in range(0, nsweeps, K):
        for g in range(world):
            plans[g].sweeps(bs[g], us[g], k, K)
        staged = []
        for g in range(world):
            for m in msgs[g]:
                staged.append((m["peer"], g, us[g][m["send_row"]:m["send_row"] + m["rows"]].clone()))
        for peer, src, blk in staged:
            m = [x for x in msgs[peer] if x["peer"] == src][0]
            us[peer][m["recv_row"]:m["recv_row"] + m["rows"]] = blk
    field = torch.cat([us[g][H:-H] for g in range(world)]).cpu().numpy()
    s_ = oracle.schedule(stencil, nx, ny, 1e-8)
    uo = oracle.sweeps(stencil, u0, oracle.rhs_to_g(stencil, h, b), s_["w"], 0, nsweeps)
    assert np.array_equal(field, uo[r:-r])
    for p_ in plans:
        p_.close()


def test_external_halo_plan_refuses_solve():
    u0, b, h = inputs.test_problem(64, 64, 1)
    with cjm.Plan(9, 64, 64, h, 1e-8, world_size=2, rank=0, external_halo=1, temporal_k=1) as plan:
        y0, nyl = plan.y0, plan.ny_local
        with pytest.raises(cjm.CJMError) as e:
            plan.solve(torch.from_numpy(b[:nyl].copy()).cuda(),
                       torch.from_numpy(u0[:nyl + 2].copy()).cuda())
        assert e.value.name == "CJM_ERR_UNSUPPORTED"


def test_external_halo_sweeps_limited_to_one_launch():
    """external_halo plans: the caller refreshes the halos between calls, so a
    call may apply at most temporal_k sweeps (one launch)."""
    u0, b, h = inputs.test_problem(64, 64, 1)
    with cjm.Plan(9, 64, 64, h, 1e-8, world_size=2, rank=0, external_halo=1, temporal_k=2) as plan:
        nyl, H = plan.ny_local, plan.ghost_rows
        ud = torch.from_numpy(np.pad(u0, ((H - 1, H - 1), (0, 0)))[:nyl + 2 * H].copy()).cuda()
        bd = torch.from_numpy(np.pad(b, ((H, H), (0, 0)))[:nyl + 2 * H].copy()).cuda()
        plan.sweeps(bd, ud, 0, 2)
        with pytest.raises(cjm.CJMError) as e:
            plan.sweeps(bd, ud, 0, 3)
        assert e.value.name == "CJM_ERR_INVALID_ARG"


def test_target_grid_in_8_slabs_deep_halos_bitwise():
    """The 8-GPU strong-scaling layout of the north_star target on one GPU:
    16384^2 in 8 row slabs of 2048 rows, K = 4 fused sweeps per launch with
    H = 4 deep halos and the band-split overlap schedule (external_halo plans,
    halos moved with device copies after every launch), two launches: bitwise
    equal to the whole-domain default plan."""
    n, world, K, launches = 16384, 8, 4, 2
    free = torch.cuda.mem_get_info()[0]
    assert free > 40e9, "a B200 holds the whole grid plus the slabs"
    u0, b, h = inputs.test_problem(n, n, 1, init="random", seed=83)
    plans = [cjm.Plan(9, n, n, h, 1e-8, world_size=world, rank=g, external_halo=1, temporal_k=K,
                      band_split=1) for g in range(world)]
    H = plans[0].ghost_rows
    assert H == K and plans[0].info()["temporal_k"] == K
    u_pad = np.pad(u0, ((H - 1, H - 1), (0, 0)))
    b_pad = np.pad(b, ((H, H), (0, 0)))
    us, bs, msgs = [], [], []
    for g in range(world):
        y0, nyl = cjm.cjm_slab(n, world, g)
        us.append(torch.from_numpy(u_pad[y0:y0 + nyl + 2 * H].copy()).cuda())
        bs.append(torch.from_numpy(b_pad[y0:y0 + nyl + 2 * H].copy()).cuda())
        msgs.append(cjm.cjm_halo_plan(n, H, world, g))
    for k in range(launches):
        for g in range(world):
            plans[g].sweeps(bs[g], us[g], k * K, K)
        staged = []
        for g in range(world):
            for m in msgs[g]:
                staged.append((m["peer"], g, us[g][m["send_row"]:m["send_row"] + m["rows"]].clone()))
        for peer, src, blk in staged:
            m = [x for x in msgs[peer] if x["peer"] == src][0]
            us[peer][m["recv_row"]:m["recv_row"] + m["rows"]] = blk
    field = torch.cat([us[g][H:-H] for g in range(world)]).cpu().numpy()
    for p_ in plans:
        p_.close()
    del us, bs
    with cjm.Plan(9, n, n, h, 1e-8) as whole:
        ud = torch.from_numpy(u0).cuda()
        whole.sweeps(torch.from_numpy(b).cuda(), ud, 0, launches * K)
        ref = ud.cpu().numpy()
    assert np.array_equal(field, ref[1:-1])
