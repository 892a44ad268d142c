"""Repeated-run stress test of the TMA ring (slot reuse across the generic
and async proxies).  A shallow ring (2 stages) and the cheapest consumer
(K = 1) make a missing cross-proxy fence show up as a non-deterministic
wrong value within a few dozen runs (it did: 35 of 200 runs before
fence.proxy.async was added).  The shipped configuration (one CTA of 11
consumer warps per SM, K = 4, 20% dynamic work items from the device counter)
runs too.  Every run must equal the oracle."""
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


@pytest.mark.parametrize("variant,K,stages,warps", [(7, 1, 2, 4), (7, 2, 3, 5), (7, 3, 3, 0), (3, 1, 2, 0),
                                                    (7, 4, 3, 11), (7, 4, 0, 0)])
def test_ring_reuse_is_race_free(variant, K, stages, warps):
    n, cnt, trials = 1024, 16, 60
    u0, b, h = inputs.test_problem(n, n, 1, init="random")
    s = oracle.schedule(5, n, n, 1e-8)
    ref = oracle.sweeps(5, u0, oracle.rhs_to_g(5, h, b), s["w"], 0, cnt)
    bd = torch.from_numpy(b).cuda()
    bad = 0
    kw = dict(warps=warps) if variant == 7 else {}
    with cjm.Plan(5, n, n, h, 1e-8, temporal_k=K, variant=variant, stages=stages, resident=-1,
                  **kw) as plan:
        for _ in range(trials):
            ud = torch.from_numpy(u0.copy()).cuda()
            plan.sweeps(bd, ud, 0, cnt)
            bad += not np.array_equal(ud.cpu().numpy(), ref)
    assert bad == 0, f"{bad} of {trials} runs differ from the oracle"


def test_resident_handshakes_are_race_free():
    n, cnt, trials = 1024, 64, 30
    u0, b, h = inputs.test_problem(n, n, 1, init="random")
    s = oracle.schedule(9, n, n, 1e-8)
    ref = oracle.sweeps(9, u0, oracle.rhs_to_g(9, h, b), s["w"], 0, cnt)
    bd = torch.from_numpy(b).cuda()
    bad = 0
    with cjm.Plan(9, n, n, h, 1e-8, resident=1) as plan:
        for _ in range(trials):
            ud = torch.from_numpy(u0.copy()).cuda()
            plan.sweeps(bd, ud, 0, cnt)
            bad += not np.array_equal(ud.cpu().numpy(), ref)
    assert bad == 0, f"{bad} of {trials} runs differ from the oracle"


@pytest.mark.parametrize("stencil,n", [(9, 4096), (17, 4096)])
def test_shipped_default_configuration_is_race_free(stencil, n):
    """The default plan of a grid large enough for dynamic work items (9-point:
    K = 4, one CTA of 11 consumer warps per SM; 17-point: K = 3), repeated:
    every run bitwise equal to the oracle."""
    r = oracle.reach(stencil)
    cnt, trials = 9, 12
    u0, b, h = inputs.test_problem(n, n, r, init="random", seed=41)
    s = oracle.schedule(stencil, n, n, 1e-8)
    ref = oracle.sweeps(stencil, u0, oracle.rhs_to_g(stencil, h, b), s["w"], 7, cnt)
    bd = torch.from_numpy(b).cuda()
    bad = 0
    with cjm.Plan(stencil, n, n, h, 1e-8) as plan:
        info = plan.info()
        assert info["variant"] == 7 and info["temporal_k"] == (4 if stencil == 9 else 3)
        if stencil == 9:
            assert info["warps"] == 11
        for _ in range(trials):
            ud = torch.from_numpy(u0.copy()).cuda()
            plan.sweeps(bd, ud, 7, cnt)
            bad += not np.array_equal(ud.cpu().numpy(), ref)
    assert bad == 0, f"{bad} of {trials} runs differ from the oracle"
