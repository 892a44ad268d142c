"""The C ABI used from plain C (tests/c_abi_demo.c compiled with gcc against
include/cjm.h and libcjm.so): no Python binding, no torch.  The host-only
entry points are checked here against the oracle's independent scheduler;
the device solve (-m gpu) against the oracle's stored solve."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

import oracle
from conftest import ROOT, has_gpu
from paper_1705_00103_b200 import cjm

SRC = os.path.join(ROOT, "tests", "c_abi_demo.c")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cabi") / "c_abi_demo")
    libdir = os.path.dirname(os.path.abspath(cjm.LIB_PATH))   # CJM_LIB may name a measurement build
    subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", SRC, "-I",
                           os.path.join(ROOT, "include"), "-L", libdir,
                           "-l:" + os.path.basename(cjm.LIB_PATH),
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    return exe


def _run(exe, *args):
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    return out.returncode, [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]


def test_host_entry_points_from_c(demo):
    rc, lines = _run(demo, "host")
    assert rc == 0
    sched, cap, geo = lines
    o = oracle.schedule(9, 64, 64, 1e-8)
    assert sched["version"] == cjm.cjm_version()
    assert float.fromhex(sched["kappa_min"]) == o["kappa_min"]
    assert float.fromhex(sched["kappa_max"]) == o["kappa_max"]
    assert sched["m_min"] == o["m_min"] and sched["P"] == o["P"]
    assert [sched["t0"], sched["t1"]] == o["t"][:2].tolist()
    assert float.fromhex(sched["w0"]) == o["w"][0] and float.fromhex(sched["wlast"]) == o["w"][-1]
    assert cap["status"] == "CJM_ERR_INVALID_ARG"
    assert geo["status"] == "CJM_OK" and geo["ld"] == geo["ld_layout"] and geo["col0"] == 8
    assert (geo["y0"], geo["ny_local"]) == (3 * 2048, 2048)
    assert geo["nxfers"] == 2 and geo["peer0"] == 2
    assert geo["send0"] == 4 * geo["ld"] and geo["recv0"] == 0 and geo["count0"] == 4 * geo["ld"]


@pytest.mark.gpu
def test_solve_host_from_c_matches_oracle(demo):
    """cjm_solve_host called from C on the paper's test problem (64^2, 9-point,
    tol 1e-8): the oracle's iteration count and its field, bitwise, on the
    inputs the C program built (it prints them)."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    rc, lines = _run(demo, "solve", "64")
    assert rc == 0, lines
    inp, solve, field = lines
    assert solve["status"] == "CJM_OK"
    h = float.fromhex(inp["h"])
    u0 = np.array([float.fromhex(v) for v in inp["u0"]]).reshape(66, 66)
    b = np.array([float.fromhex(v) for v in inp["b"]]).reshape(64, 64)
    uo, ro = oracle.solve(9, h, 1e-8, b, u0)
    assert solve["iterations"] == ro["iterations"]
    got = np.array([float.fromhex(v) for v in field["values"]]).reshape(64, 64)
    want = uo[1:-1, 1:-1]
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
    assert np.array_equal(got, want)
    assert solve["h2d_bytes"] == 66 * 66 * 8 + 64 * 64 * 8 and solve["d2h_bytes"] == 64 * 64 * 8
