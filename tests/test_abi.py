"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/cjm.h declares, its host scheduler agrees bit for bit with the
oracle's independently written scheduler, and compute entry points fail
loudly (no CPU fallback) when no GPU is present."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, has_gpu
from paper_1705_00103_b200 import cjm

HEADER = os.path.join(ROOT, "include", "cjm.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cjm_[a-z_0-9]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    L = cjm.lib()
    names = header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(cjm.EXPORTS)
    assert cjm.cjm_version() == 1


def test_library_is_sm100a():
    data = open(cjm.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


@pytest.mark.parametrize("stencil", (5, 9, 17))
@pytest.mark.parametrize("nx,ny", [(64, 64), (1024, 1024), (4096, 4096), (8192, 8192),
                                   (16384, 16384), (4096, 32768), (300, 77)])
def test_scheduler_bitwise_equals_oracle(stencil, nx, ny):
    s = cjm.cjm_schedule(stencil, nx, ny, 1e-8)
    o = oracle.schedule(stencil, nx, ny, 1e-8)
    assert s["kappa_min"] == o["kappa_min"] and s["kappa_max"] == o["kappa_max"]
    assert s["m_min"] == o["m_min"] and s["P"] == o["P"]
    assert np.array_equal(s["t"], o["t"])
    assert np.array_equal(s["w"], o["w"])


@pytest.mark.parametrize("stencil,nx,ny", [(9, 64, 64), (17, 1024, 1024), (5, 4096, 4096), (9, 16384, 16384)])
def test_scheduler_lebedev2_bitwise_equals_oracle(stencil, nx, ny):
    s = cjm.cjm_schedule(stencil, nx, ny, 1e-8, order=cjm.ORDER_LEBEDEV2)
    o = oracle.schedule(stencil, nx, ny, 1e-8, order="lebedev2")
    assert s["P"] == o["P"] and s["m_min"] == o["m_min"]
    assert np.array_equal(s["t"], o["t"]) and np.array_equal(s["w"], o["w"])


def test_buffer_layout_and_halo_xfers():
    """The NCCL exchange's element-level transfers are cjm_halo_plan's rows in
    the internal layout (whole rows of pitch ld)."""
    for nx in (1, 37, 4096, 16384):
        ld, c0 = cjm.cjm_buffer_layout(nx)
        assert ld % 32 == 0 and ld >= nx + 2 * c0 and c0 == 8
    for ny, depth, world in [(100, 1, 4), (4096, 4, 8), (16384, 8, 2)]:
        for rank in range(world):
            xs, ld = cjm.cjm_halo_xfers(4096, ny, depth, world, rank)
            msgs = cjm.cjm_halo_plan(ny, depth, world, rank)
            assert len(xs) == len(msgs)
            for x, m in zip(xs, msgs):
                assert x["peer"] == m["peer"] and x["count"] == m["rows"] * ld
                assert x["send_off"] == m["send_row"] * ld and x["recv_off"] == m["recv_row"] * ld


def test_scheduler_ascending_order_option():
    s = cjm.cjm_schedule(9, 64, 64, 1e-8, order=cjm.ORDER_ASCENDING)
    assert np.all(np.diff(s["w"]) > 0)
    o = oracle.schedule(9, 64, 64, 1e-8)
    assert np.array_equal(np.sort(s["w"]), np.sort(o["w"]))


@pytest.mark.parametrize("args", [(7, 64, 64, 1e-8), (9, 3, 64, 1e-8), (9, 64, 64, 0.0),
                                  (9, 64, 64, 1.0), (9, 64, 64, float("nan"))])
def test_scheduler_invalid_args(args):
    with pytest.raises(cjm.CJMError) as e:
        cjm.cjm_schedule(*args)
    assert e.value.name == "CJM_ERR_INVALID_ARG"


@pytest.mark.parametrize("ny,world", [(4096, 1), (4096, 8), (8192, 3), (100, 7), (32768, 8)])
def test_slab_partition(ny, world):
    rows = []
    for g in range(world):
        y0, n = cjm.cjm_slab(ny, world, g)
        assert y0 == g * ny // world and n == (g + 1) * ny // world - y0
        rows += list(range(y0, y0 + n))
    assert rows == list(range(ny))


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_plan_fails_loudly_without_gpu():
    with pytest.raises(cjm.CJMError) as e:
        cjm.Plan(9, 64, 64, 1 / 65, 1e-8)
    assert e.value.name == "CJM_ERR_CUDA"


def test_plan_rejects_bad_arguments_before_touching_the_device():
    for kw in [dict(stencil=9, nx=64, ny=64, h=-1.0, tol=1e-8),
               dict(stencil=11, nx=64, ny=64, h=0.1, tol=1e-8),
               dict(stencil=9, nx=64, ny=2, h=0.1, tol=1e-8),
               dict(stencil=9, nx=64, ny=64, h=0.1, tol=2.0)]:
        with pytest.raises(cjm.CJMError) as e:
            cjm.Plan(**kw)
        assert e.value.name == "CJM_ERR_INVALID_ARG"
    with pytest.raises(cjm.CJMError) as e:
        cjm.Plan(9, 64, 64, 0.1, 1e-8, bc=1)
    assert e.value.name == "CJM_ERR_UNSUPPORTED"
    with pytest.raises(cjm.CJMError) as e:   # world > 1 without an NCCL id
        cjm.Plan(9, 64, 64, 0.1, 1e-8, world_size=2, rank=0)
    assert e.value.name == "CJM_ERR_INVALID_ARG"


def test_no_shared_code_between_oracle_and_product():
    pkg = os.path.join(ROOT, "paper_1705_00103_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), f
                assert "cjm_oracle" not in src and "liboracle" not in src, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_1705_00103_b200", src, re.M), f
            assert "#include" not in src or "cjm.h" not in src, f
