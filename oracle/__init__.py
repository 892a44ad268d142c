"""ctypes front-end of the CPU oracle (oracle/cjm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_1705_00103_b200`` never imports it, and
this module never imports the product package: the two share no code.

Every function is a thin marshalling layer over the C oracle; the arithmetic
(and the paper citations for it) lives in ``cjm_oracle.c``.

Parity status: every function below is pinned by -m "not gpu" tests
(tests/test_oracle_pins.py); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cjm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_cjm.so")

# -ffp-contract=off: no fused multiply-add other than the explicit fma() calls
# (DESIGN R6).  -mfma only makes fma() an instruction instead of a libm call;
# both are correctly rounded.
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
          "-fno-fast-math", "-mfma", "-std=c11", "-D_GNU_SOURCE", "-Wall"]

STATUS = {0: "OK", 1: "INVALID", 3: "NOT_CONVERGED", 4: "DIVERGED",
          5: "STAGNATED", 8: "OOM"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Report(C.Structure):
    _fields_ = [("iterations", C.c_longlong), ("cycles", C.c_int), ("status", C.c_int),
                ("cycle_len", C.c_longlong), ("m_min", C.c_longlong),
                ("kappa_min", C.c_double), ("kappa_max", C.c_double),
                ("r0_l2", C.c_double), ("r0_linf", C.c_double),
                ("r_l2", C.c_double), ("r_linf", C.c_double)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["status"] = STATUS.get(self.status, str(self.status))
        return d


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        L.oracle_reach.argtypes = [C.c_int]
        L.oracle_bounds.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp]
        L.oracle_m_min.argtypes = [C.c_double, C.c_double, C.c_double]
        L.oracle_m_min.restype = C.c_long
        L.oracle_cycle_len.argtypes = [C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.oracle_cycle_len.restype = C.c_long
        L.oracle_cycle_len_pow2.argtypes = [C.c_long, C.POINTER(C.c_int)]
        L.oracle_cycle_len_pow2.restype = C.c_long
        L.oracle_ordering.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_long)]
        L.oracle_weights.argtypes = [C.c_double, C.c_double, C.c_long, C.POINTER(C.c_long), dp]
        L.oracle_gscale.argtypes = [C.c_int, C.c_double]
        L.oracle_gscale.restype = C.c_double
        L.oracle_rhs_to_g.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, dp, C.c_long, dp, C.c_long]
        L.oracle_sweep.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, dp, C.c_long,
                                   C.c_double, dp, C.c_long]
        L.oracle_delta_norms.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, dp, C.c_long, dp, dp]
        L.oracle_residual.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, dp, C.c_long,
                                      dp, C.c_long, dp, dp]
        L.oracle_solve.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                   dp, C.c_long, dp, C.c_long, dp, C.c_long, C.POINTER(Report),
                                   C.c_int]
        L.oracle_sweeps.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, dp, C.c_long, dp,
                                    C.c_long, C.c_long, C.c_long, C.c_int]
        L.oracle_odd_closure.argtypes = [C.c_int, C.c_int, dp, C.c_long]
        L.oracle_mask_sweep.argtypes = [C.c_int, C.c_int, dp, C.c_long, dp, dp, dp, dp, dp, C.c_long,
                                        dp, C.c_long, C.c_double, dp, C.c_long]
        L.oracle_mask_residual.argtypes = [C.c_int, C.c_int, dp, C.c_long, dp, dp, dp, dp, dp, C.c_long,
                                           dp, C.c_long, dp, dp]
        L.oracle_mask_solve.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, dp, C.c_long, dp, C.c_long,
                                        C.c_double, C.c_double, C.c_double, C.c_int, dp, C.c_long,
                                        C.POINTER(Report)]
        pp = C.POINTER(C.c_void_p)
        L.oracle_maskn_sweep.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, pp, C.c_long, dp,
                                         C.c_long, C.c_double, dp, C.c_long]
        L.oracle_maskn_residual.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, pp, C.c_long, dp,
                                            C.c_long, dp, dp]
        L.oracle_maskn_solve.argtypes = [C.c_int, C.c_int, C.c_int, pp, C.c_long, dp, C.c_long,
                                         C.c_double, C.c_double, C.c_double, C.c_int, dp, C.c_long,
                                         C.POINTER(Report)]
        L.oracle_num_threads.restype = C.c_int
        L.oracle_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def reach(stencil: int) -> int:
    return lib().oracle_reach(stencil)


def bounds(stencil: int, nx: int, ny: int) -> tuple[float, float]:
    a, b = C.c_double(), C.c_double()
    if lib().oracle_bounds(stencil, nx, ny, C.byref(a), C.byref(b)):
        raise ValueError("bad stencil")
    return a.value, b.value


def m_min(kmin: float, kmax: float, tol: float) -> int:
    return int(lib().oracle_m_min(kmin, kmax, tol))


def cycle_len(m: int) -> tuple[int, int, int]:
    a, b = C.c_int(), C.c_int()
    P = lib().oracle_cycle_len(m, C.byref(a), C.byref(b))
    return int(P), a.value, b.value


def cycle_len_pow2(m: int) -> tuple[int, int]:
    a = C.c_int()
    P = lib().oracle_cycle_len_pow2(m, C.byref(a))
    return int(P), a.value


def ordering(a: int, b: int) -> np.ndarray:
    P = 2 ** a * 3 ** b
    t = (C.c_long * P)()
    lib().oracle_ordering(a, b, t)
    return np.frombuffer(t, dtype=np.int64).copy()


def weights(kmin: float, kmax: float, t: np.ndarray) -> np.ndarray:
    t = np.ascontiguousarray(t, dtype=np.int64)
    w = np.empty(len(t), dtype=np.float64)
    lib().oracle_weights(kmin, kmax, len(t), t.ctypes.data_as(C.POINTER(C.c_long)), _dp(w))
    return w


def schedule(stencil: int, nx: int, ny: int, tol: float, order: str = "lebedev23") -> dict:
    """Steps 1-3 in one call: bounds, M, P=2^a3^b (order "lebedev2": P=2^a),
    ordering t, weights w."""
    kmin, kmax = bounds(stencil, nx, ny)
    m = m_min(kmin, kmax, tol)
    if order == "lebedev2":
        P, a = cycle_len_pow2(m)
        b = 0
    elif order == "lebedev23":
        P, a, b = cycle_len(m)
    else:
        raise ValueError(order)
    t = ordering(a, b)
    return dict(kappa_min=kmin, kappa_max=kmax, m_min=m, P=P, a=a, b=b, t=t,
                w=weights(kmin, kmax, t))


def gscale(stencil: int, h: float) -> float:
    return lib().oracle_gscale(stencil, h)


def rhs_to_g(stencil: int, h: float, b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    g = np.empty_like(b)
    lib().oracle_rhs_to_g(stencil, nx, ny, h, _dp(b), nx, _dp(g), nx)
    return g


def sweep(stencil: int, u: np.ndarray, g: np.ndarray, w: float) -> np.ndarray:
    """One weighted Jacobi sweep; u carries its r ghost rings, g = D^-1 b."""
    r = reach(stencil)
    u = np.ascontiguousarray(u, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    ny, nx = u.shape[0] - 2 * r, u.shape[1] - 2 * r
    assert g.shape == (ny, nx)
    out = u.copy()
    lib().oracle_sweep(stencil, nx, ny, _dp(u), u.shape[1], _dp(g), nx, w, _dp(out), u.shape[1])
    return out


CLOSURES = {"dirichlet": 0, "odd": 1}


def odd_closure(u: np.ndarray) -> np.ndarray:
    """A copy of the 17-point field u (2 ghost rings) with its outer ring set
    by odd reflection through the boundary (oracle_odd_closure, DESIGN R12)."""
    out = np.array(u, dtype=np.float64, order="C", copy=True)
    ny, nx = out.shape[0] - 4, out.shape[1] - 4
    lib().oracle_odd_closure(nx, ny, _dp(out), out.shape[1])
    return out


def sweeps(stencil: int, u: np.ndarray, g: np.ndarray, w: np.ndarray, first: int,
           count: int, closure: str = "dirichlet") -> np.ndarray:
    """`count` scheduled sweeps (weight w[(first+k) mod P] at sweep k);
    closure="odd" (17-point): outer ghost ring reflected before every sweep."""
    r = reach(stencil)
    out = np.array(u, dtype=np.float64, order="C", copy=True)
    g = np.ascontiguousarray(g, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    ny, nx = out.shape[0] - 2 * r, out.shape[1] - 2 * r
    st = lib().oracle_sweeps(stencil, nx, ny, _dp(out), out.shape[1], _dp(g), nx, _dp(w), len(w),
                             first, count, CLOSURES[closure])
    if st != 0:
        raise ValueError(f"oracle_sweeps: status {st}")
    return out


def delta_norms(stencil: int, u: np.ndarray, g: np.ndarray) -> tuple[float, float]:
    r = reach(stencil)
    u = np.ascontiguousarray(u, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    ny, nx = u.shape[0] - 2 * r, u.shape[1] - 2 * r
    s, m = C.c_double(), C.c_double()
    lib().oracle_delta_norms(stencil, nx, ny, _dp(u), u.shape[1], _dp(g), nx, C.byref(s), C.byref(m))
    return s.value, m.value


def residual(stencil: int, h: float, b: np.ndarray, u: np.ndarray) -> tuple[float, float]:
    """(||b - Delta_h u||_2, ||b - Delta_h u||_inf) over the interior."""
    r = reach(stencil)
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    l2, li = C.c_double(), C.c_double()
    lib().oracle_residual(stencil, nx, ny, h, _dp(b), nx, _dp(u), u.shape[1], C.byref(l2), C.byref(li))
    return l2.value, li.value


def solve(stencil: int, h: float, tol: float, b: np.ndarray, u0: np.ndarray,
          max_cycles: int = 8, weights_override: np.ndarray | None = None,
          closure: str = "dirichlet"):
    """Full CJM solve.  Returns (u, report dict); u0 is not modified.
    closure="odd" (17-point): the outer ghost ring by odd reflection,
    recomputed before every sweep and residual (DESIGN R12)."""
    u = np.array(u0, dtype=np.float64, order="C", copy=True)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    rep = Report()
    if weights_override is not None:
        wo = np.ascontiguousarray(weights_override, dtype=np.float64)
        wp, wl = _dp(wo), len(wo)
    else:
        wo, wp, wl = None, None, 0
    lib().oracle_solve(stencil, nx, ny, h, tol, max_cycles, _dp(b), nx, _dp(u), u.shape[1],
                       wp, wl, C.byref(rep), CLOSURES[closure])
    return u, rep.as_dict()


def _mask_args(mask):
    cs = [np.ascontiguousarray(mask[k], dtype=np.float64) for k in ("W", "E", "S", "N", "C")]
    return cs, [_dp(c) for c in cs]


def mask_sweep(mask: dict, u: np.ndarray, b: np.ndarray, w: float) -> np.ndarray:
    """One weighted Jacobi sweep with a generic 5-point mask (dict of per-node
    coefficient arrays W, E, S, N, C, each ny x nx); u has one ghost ring."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, ps = _mask_args(mask)
    out = u.copy()
    lib().oracle_mask_sweep(nx, ny, _dp(u), u.shape[1], *ps, nx, _dp(b), nx, w, _dp(out), u.shape[1])
    return out


def mask_residual(mask: dict, u: np.ndarray, b: np.ndarray) -> tuple[float, float]:
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, ps = _mask_args(mask)
    l2, li = C.c_double(), C.c_double()
    lib().oracle_mask_residual(nx, ny, _dp(u), u.shape[1], *ps, nx, _dp(b), nx, C.byref(l2), C.byref(li))
    return l2.value, li.value


def mask_solve(mask: dict, b: np.ndarray, u0: np.ndarray, kmin: float, kmax: float, tol: float,
               max_cycles: int = 8):
    u = np.array(u0, dtype=np.float64, order="C", copy=True)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, ps = _mask_args(mask)
    rep = Report()
    lib().oracle_mask_solve(nx, ny, *ps, nx, _dp(b), nx, kmin, kmax, tol, max_cycles, _dp(u), u.shape[1],
                            C.byref(rep))
    return u, rep.as_dict()


def _maskn_args(planes):
    """planes: list of (2m+1)^2 per-node coefficient arrays (ny x nx) or None."""
    keep = [None if c is None else np.ascontiguousarray(c, dtype=np.float64) for c in planes]
    arr = (C.c_void_p * len(keep))(*[None if c is None else c.ctypes.data for c in keep])
    return keep, arr


def maskn_radius(planes) -> int:
    m = {9: 1, 25: 2}.get(len(planes))
    if m is None:
        raise ValueError("a generic mask has 9 (m = 1) or 25 (m = 2) planes")
    return m


def maskn_sweep(planes, u: np.ndarray, b: np.ndarray, w: float) -> np.ndarray:
    """One weighted Jacobi sweep with a generic (2m+1)^2 mask (planes in
    row-major mask order, q = (dy+m)(2m+1) + (dx+m); None = absent); u has m
    ghost rings."""
    m = maskn_radius(planes)
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, arr = _maskn_args(planes)
    out = u.copy()
    lib().oracle_maskn_sweep(m, nx, ny, _dp(u), u.shape[1], arr, nx, _dp(b), nx, w, _dp(out), u.shape[1])
    return out


def maskn_residual(planes, u: np.ndarray, b: np.ndarray) -> tuple[float, float]:
    m = maskn_radius(planes)
    u = np.ascontiguousarray(u, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, arr = _maskn_args(planes)
    l2, li = C.c_double(), C.c_double()
    lib().oracle_maskn_residual(m, nx, ny, _dp(u), u.shape[1], arr, nx, _dp(b), nx, C.byref(l2),
                                C.byref(li))
    return l2.value, li.value


def maskn_solve(planes, b: np.ndarray, u0: np.ndarray, kmin: float, kmax: float, tol: float,
                max_cycles: int = 8):
    m = maskn_radius(planes)
    u = np.array(u0, dtype=np.float64, order="C", copy=True)
    b = np.ascontiguousarray(b, dtype=np.float64)
    ny, nx = b.shape
    keep, arr = _maskn_args(planes)
    rep = Report()
    lib().oracle_maskn_solve(m, nx, ny, arr, nx, _dp(b), nx, kmin, kmax, tol, max_cycles, _dp(u),
                             u.shape[1], C.byref(rep))
    return u, rep.as_dict()


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(n)
