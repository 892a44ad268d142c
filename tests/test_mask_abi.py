"""CPU-only checks of the generic-mask entry points of the C ABI (NEXT-4):
the host spectral-bound estimator cjm_mask_bounds against closed forms and
dense eigenvalues, and argument validation of cjm_plan_mask before any
device work."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_1705_00103_b200 import cjm, masks
from test_oracle_masks import _dense_bounds


@pytest.mark.parametrize("nx,ny", [(20, 20), (37, 12), (64, 64)])
def test_mask_bounds_cartesian_closed_form(nx, ny):
    """Cartesian mask = the 5-point stencil: eigenvalues of D^-1 A are
    sin^2(k pi/2Nx) + sin^2(l pi/2Ny) (P:86, S:252 with N = n + 1, DESIGN R1):
    kappa_min = sin^2(pi/2Nx) + sin^2(pi/2Ny), kappa_max = 2 - kappa_min."""
    h = 1.0 / (nx + 1)
    kmin, kmax = cjm.cjm_mask_bounds(masks.cartesian(nx, ny, h), iters=50)
    want = math.sin(math.pi / (2 * (nx + 1))) ** 2 + math.sin(math.pi / (2 * (ny + 1))) ** 2
    assert kmin == pytest.approx(want, rel=1e-10)
    assert kmax == pytest.approx(2.0 - want, rel=1e-13)


@pytest.mark.parametrize("kind", ["polar", "bipolar"])
def test_mask_bounds_match_dense_eigenvalues(kind):
    mk = (masks.polar_problem if kind == "polar" else masks.bipolar_problem)(24, 20)[0]
    lo, hi = _dense_bounds(mk)
    assert lo + hi == pytest.approx(2.0, abs=1e-12)        # bipartite symmetry about 1
    kmin, kmax = cjm.cjm_mask_bounds(mk, iters=4000)
    assert kmin == pytest.approx(lo, rel=1e-6) and kmin >= lo * (1 - 1e-12)
    assert kmax == pytest.approx(hi, rel=1e-9)


def test_mask_bounds_reject_bad_masks():
    mk = masks.cartesian(8, 8, 0.1)
    bad = dict(mk)
    bad["C"] = mk["C"].copy()
    bad["C"][3, 4] = 0.0
    with pytest.raises(cjm.CJMError) as e:
        cjm.cjm_mask_bounds(bad)
    assert e.value.name == "CJM_ERR_INVALID_ARG"
    indef = dict(mk)
    indef["C"] = mk["C"] * 0.4            # a_q = 0.625: rho(N) ~ 2.5 > 1, D^-1 A indefinite
    with pytest.raises(cjm.CJMError):
        cjm.cjm_mask_bounds(indef)


def test_plan_mask_rejects_bad_arguments_before_touching_the_device():
    for args in [(64, 64, 0.0, 1.0, 1e-8), (64, 64, 0.5, 0.4, 1e-8), (64, 64, 0.1, float("inf"), 1e-8),
                 (3, 64, 0.1, 1.9, 1e-8), (64, 64, 0.1, 1.9, 0.0)]:
        with pytest.raises(cjm.CJMError) as e:
            cjm.MaskPlan(*args)
        assert e.value.name == "CJM_ERR_INVALID_ARG"
    with pytest.raises(cjm.CJMError) as e:
        cjm.MaskPlan(64, 64, 0.1, 1.9, 1e-8, world_size=2, rank=0)
    assert e.value.name == "CJM_ERR_UNSUPPORTED"
    with pytest.raises(cjm.CJMError) as e:                     # masks only via cjm_plan_mask
        cjm.Plan(cjm.STENCIL_MASK, 64, 64, 0.1, 1e-8)
    assert e.value.name == "CJM_ERR_INVALID_ARG"



@pytest.mark.parametrize("m,nx,ny", [(1, 12, 10), (2, 11, 13)])
@pytest.mark.parametrize("kind", ("cartesian", "symmetric"))
def test_mask_bounds_n_match_dense_eigenvalues(m, nx, ny, kind):
    """cjm_mask_bounds_n (host power iterations, no GPU) vs the dense spectrum
    of D^-1 A for square masks (SURVEY A14's numeric fallback)."""
    import numpy as np
    from paper_1705_00103_b200 import masks
    if kind == "cartesian":
        planes = masks.cartesian_n(9 if m == 1 else 17, nx, ny, 1.0 / (nx + 1))
    else:
        planes = masks.symmetric_n(m, nx, ny, seed=7)
    s = 2 * m + 1
    n = nx * ny
    B = np.zeros((n, n))
    cc = planes[m * s + m]
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            B[k, k] = 1.0
            for q, c in enumerate(planes):
                if c is None or q == m * s + m:
                    continue
                ii, jj = i + q % s - m, j + q // s - m
                if 0 <= ii < nx and 0 <= jj < ny:
                    B[k, jj * nx + ii] = c[j, i] / cc[j, i]
    ev = np.linalg.eigvals(B)
    assert np.max(np.abs(ev.imag)) < 1e-9
    lo, hi = float(np.min(ev.real)), float(np.max(ev.real))
    kmin, kmax = cjm.cjm_mask_bounds_n(planes, iters=20000)
    assert kmax == pytest.approx(hi, rel=1e-6)
    assert kmin == pytest.approx(lo, rel=1e-3)
    assert kmin >= lo * (1 - 1e-9) and kmax <= hi * (1 + 1e-9)   # from inside the spectrum


def test_mask_bounds_n_rejects_mismatched_planes():
    """Every present plane must have the centre plane's shape (the C power
    iteration would read past a smaller host buffer), and the centre plane
    is required."""
    import numpy as np
    n = 8
    planes = [None] * 9
    planes[4] = np.full((n, n), -20.0 / 6.0)
    for q in (1, 3, 5, 7):
        planes[q] = np.full((n, n), 4.0 / 6.0)
    planes[1] = np.full((n - 1, n), 4.0 / 6.0)
    with pytest.raises(ValueError):
        cjm.cjm_mask_bounds_n(planes)
    planes[1] = np.full((n, n), 4.0 / 6.0)
    planes[4] = None
    with pytest.raises(ValueError):
        cjm.cjm_mask_bounds_n(planes)
