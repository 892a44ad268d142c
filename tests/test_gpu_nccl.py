"""The NCCL data plane on one GPU.

A plan given an NCCL unique id with world_size = 1 creates a ONE-rank
communicator (ncclCommInitRank) and runs the multi-GPU schedule of the
library: hot sweeps split into boundary bands + interior band, the halo
exchange forked onto the plan's comm stream and joined back (captured in the
CUDA graphs; with one rank the NCCL group has no peers), the residual
reduction allreduced (sum, max) through NCCL, the real-error reduction
allreduced, and the communicator cache.  Everything must be bitwise equal to
the oracle.  (Two ranks cannot share one GPU in an NCCL communicator; the
transfers of more ranks are covered by tests/test_multirank.py on gloo, which
executes the library's own transfer list, cjm_halo_xfers.)
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("stencil,n,K", [(9, 300, 0), (9, 1030, 4), (17, 257, 3), (5, 200, 1)])
def test_one_rank_nccl_solve_bitwise(stencil, n, K):
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=61)
    uo, ro = oracle.solve(stencil, h, 1e-8, b, u0)
    nid = cjm.cjm_get_nccl_id()
    with cjm.Plan(stencil, n, n, h, 1e-8, nccl_id=nid, world_size=1, rank=0, temporal_k=K) as plan:
        info = plan.info()
        assert info["comm_nranks"] == 1 and info["comm_rank"] == 0
        assert info["resident"] == 0            # the NCCL schedule, not the resident kernel
        ud = dev(u0)
        rep = plan.solve(dev(b), ud)
    assert rep["status"] == "CJM_OK" and rep["iterations"] == ro["iterations"]
    assert rep["comm_nranks"] == 1
    # band split: 3 launches per hot step (two boundary bands + interior)
    assert rep["kernel_launches"] >= 3 * rep["hot_launches"]
    assert rep["r0_l2"] == pytest.approx(ro["r0_l2"], rel=1e-12)
    got = ud.cpu().numpy()
    assert np.array_equal(got[r:-r, r:-r], uo[r:-r, r:-r])


def test_one_rank_nccl_residual_sweeps_and_real_error():
    n, r = 257, 1
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=67)
    nid = cjm.cjm_get_nccl_id()
    with cjm.Plan(9, n, n, h, 1e-8, nccl_id=nid, world_size=1, rank=0) as plan:
        l2, li = plan.residual(dev(b), dev(u0))
        ol2, oli = oracle.residual(9, h, b, u0)
        assert l2 == pytest.approx(ol2, rel=1e-12) and li == oli
        w = plan.info()["weights"]
        ud = dev(u0)
        plan.sweeps(dev(b), ud, 11, 23)
        want = oracle.sweeps(9, u0, oracle.rhs_to_g(9, h, b), w, 11, 23)
        assert np.array_equal(ud.cpu().numpy(), want)
        ex = inputs.exact_field(n, n, r, h)
        ud = dev(inputs.test_problem(n, n, r)[0])
        rep = plan.solve_ref(dev(b), ud, dev(ex), 1e-4)
        assert rep["status"] == "CJM_OK"
        assert rep["real_error"] == np.max(np.abs(ud.cpu().numpy()[r:-r, r:-r] - ex))


def test_communicator_cache_reuse_and_live_id_conflict():
    n = 64
    u0, b, h = inputs.test_problem(n, n, 1)
    nid = cjm.cjm_get_nccl_id()
    for _ in range(3):     # the cached, idle communicator is reused (no re-initialisation)
        with cjm.Plan(9, n, n, h, 1e-8, nccl_id=nid, world_size=1, rank=0) as plan:
            rep = plan.solve(dev(b), dev(u0))
            assert rep["status"] == "CJM_OK" and rep["comm_nranks"] == 1
            with pytest.raises(cjm.CJMError) as e:   # a second LIVE plan on the same id
                cjm.Plan(9, n, n, h, 1e-8, nccl_id=nid, world_size=1, rank=0)
            assert e.value.name == "CJM_ERR_INVALID_ARG"
    cjm.cjm_pool_trim()
    # after the trim the id is unknown again: a fresh id initialises a new communicator
    with cjm.Plan(9, n, n, h, 1e-8, nccl_id=cjm.cjm_get_nccl_id(), world_size=1, rank=0) as plan:
        assert plan.info()["comm_nranks"] == 1
