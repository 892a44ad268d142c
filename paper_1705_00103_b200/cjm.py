"""Thin ctypes binding of libcjm (include/cjm.h): argument marshalling only.

Every step of the path runs in the CUDA library; this module converts torch
CUDA tensors / numpy arrays into (pointer, pitch) pairs and C structs, and
raises on error.  There is no CPU fallback: if libcjm.so is missing the import
of the library fails loudly.

Names follow the C ABI: cjm_schedule, cjm_plan, cjm_plan_info, cjm_solve,
cjm_solve_host, cjm_sweeps, cjm_residual, cjm_get_nccl_id, cjm_slab,
cjm_plan_destroy, and for generic 5-point masks (NEXT-4) cjm_plan_mask,
cjm_mask_set, cjm_mask_bounds.  The Plan / MaskPlan classes wrap a plan
handle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CJM_LIB selects a measurement build of the same library (build.build(out=...));
# there is no other implementation to fall back to.
LIB_PATH = os.environ.get("CJM_LIB") or os.path.join(HERE, "libcjm.so")

STENCIL_MASK, STENCIL_5, STENCIL_9, STENCIL_17 = 1, 5, 9, 17
BC_DIRICHLET = 0
ORDER_LEBEDEV23, ORDER_ASCENDING, ORDER_LEBEDEV2 = 0, 1, 2
METHOD_CHEBYSHEV, METHOD_JACOBI = 0, 1
CLOSURE_DIRICHLET, CLOSURE_ODD = 0, 1

STATUS = {0: "CJM_OK", 1: "CJM_ERR_INVALID_ARG", 2: "CJM_ERR_UNSUPPORTED",
          3: "CJM_ERR_NOT_CONVERGED", 4: "CJM_ERR_DIVERGED", 5: "CJM_ERR_STAGNATED",
          6: "CJM_ERR_CUDA", 7: "CJM_ERR_NCCL", 8: "CJM_ERR_OOM"}

# Symbols include/cjm.h declares (tests/test_abi.py checks the header agrees).
EXPORTS = ("cjm_default_options", "cjm_schedule", "cjm_plan", "cjm_plan_info", "cjm_solve",
           "cjm_solve_ref",
           "cjm_solve_host", "cjm_sweeps", "cjm_residual", "cjm_get_nccl_id", "cjm_slab", "cjm_halo_plan",
           "cjm_plan_destroy", "cjm_pool_trim", "cjm_status_str", "cjm_last_error", "cjm_version",
           "cjm_plan_mask", "cjm_mask_set", "cjm_mask_bounds", "cjm_plan_mask_n", "cjm_mask_set_n",
           "cjm_mask_bounds_n", "cjm_buffer_layout", "cjm_halo_xfers")


class CJMError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: {self.name}" + (f" ({detail})" if detail else ""))


class Options(C.Structure):
    _fields_ = [("max_cycles", C.c_int), ("order", C.c_int), ("method", C.c_int),
                ("jacobi_check", C.c_int), ("world_size", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("device", C.c_int), ("external_halo", C.c_int),
                ("temporal_k", C.c_int), ("variant", C.c_int),
                ("tile_w", C.c_int),
                ("ctas_per_sm", C.c_int), ("stages", C.c_int), ("graph_chunk", C.c_int),
                ("resident", C.c_int), ("band_split", C.c_int), ("warps", C.c_int),
                ("closure", C.c_int), ("chunk_rows", C.c_int)]


class HaloMsg(C.Structure):
    _fields_ = [("peer", C.c_int), ("send_row", C.c_int), ("recv_row", C.c_int), ("rows", C.c_int)]


class HaloXfer(C.Structure):
    _fields_ = [("peer", C.c_int), ("send_off", C.c_longlong), ("recv_off", C.c_longlong),
                ("count", C.c_longlong)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_longlong), ("cycles", C.c_int), ("status", C.c_int),
                ("cycle_len", C.c_longlong), ("m_min", C.c_longlong),
                ("kappa_min", C.c_double), ("kappa_max", C.c_double),
                ("r0_l2", C.c_double), ("r0_linf", C.c_double),
                ("r_l2", C.c_double), ("r_linf", C.c_double),
                ("plan_s", C.c_double), ("solve_s", C.c_double), ("sweep_s", C.c_double),
                ("sweeps_timed", C.c_longlong), ("kernel_launches", C.c_longlong),
                ("hot_launches", C.c_longlong), ("temporal_k", C.c_int), ("resident", C.c_int),
                ("ghost_rows", C.c_int), ("rhs_ghost_rows", C.c_int),
                ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double), ("real_error", C.c_double),
                ("variant", C.c_int), ("warps", C.c_int), ("stages", C.c_int), ("ctas", C.c_int),
                ("comm_nranks", C.c_int), ("comm_rank", C.c_int)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["status"] = STATUS.get(self.status, str(self.status))
        return d


_lib = None


def lib():
    """Load libcjm.so; raise (never fall back) if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    dp, vp, ll, i = C.POINTER(C.c_double), C.c_void_p, C.c_longlong, C.c_int
    L.cjm_default_options.argtypes = [C.POINTER(Options)]
    L.cjm_default_options.restype = None
    L.cjm_schedule.argtypes = [i, i, i, C.c_double, i, dp, dp, C.POINTER(ll), C.POINTER(ll),
                               C.POINTER(ll), dp, ll]
    L.cjm_plan.argtypes = [C.POINTER(vp), i, i, i, C.c_double, i, C.c_double, C.POINTER(Options)]
    L.cjm_plan_mask.argtypes = [C.POINTER(vp), i, i, C.c_double, C.c_double, C.c_double,
                                C.POINTER(Options)]
    L.cjm_mask_set.argtypes = [vp, vp, vp, vp, vp, vp, ll, vp]
    L.cjm_plan_mask_n.argtypes = [C.POINTER(vp), i, i, i, C.c_double, C.c_double, C.c_double,
                                  C.POINTER(Options)]
    L.cjm_mask_set_n.argtypes = [vp, C.POINTER(vp), ll, vp]
    L.cjm_mask_bounds_n.argtypes = [i, i, i, C.POINTER(vp), ll, i, dp, dp]
    L.cjm_mask_bounds.argtypes = [i, i, vp, vp, vp, vp, vp, ll, i, dp, dp]
    L.cjm_plan_info.argtypes = [vp, C.POINTER(Report), C.POINTER(i), C.POINTER(i), C.POINTER(i),
                                C.POINTER(dp)]
    L.cjm_solve.argtypes = [vp, vp, ll, vp, ll, vp, C.POINTER(Report)]
    L.cjm_solve_host.argtypes = [vp, vp, ll, vp, ll, vp, C.POINTER(Report)]
    L.cjm_solve_ref.argtypes = [vp, vp, ll, vp, ll, vp, ll, C.c_double, vp, C.POINTER(Report)]
    L.cjm_sweeps.argtypes = [vp, vp, ll, vp, ll, ll, ll, vp, C.POINTER(Report)]
    L.cjm_residual.argtypes = [vp, vp, ll, vp, ll, vp, dp, dp]
    L.cjm_get_nccl_id.argtypes = [vp]
    L.cjm_slab.argtypes = [i, i, i, C.POINTER(i), C.POINTER(i)]
    L.cjm_halo_plan.argtypes = [i, i, i, i, C.POINTER(HaloMsg), C.POINTER(i)]
    L.cjm_buffer_layout.argtypes = [i, C.POINTER(ll), C.POINTER(i)]
    L.cjm_halo_xfers.argtypes = [i, i, i, i, i, C.POINTER(HaloXfer), C.POINTER(i), C.POINTER(ll)]
    L.cjm_plan_destroy.argtypes = [vp]
    L.cjm_pool_trim.argtypes = [C.POINTER(ll)]
    L.cjm_status_str.argtypes = [i]
    L.cjm_status_str.restype = C.c_char_p
    L.cjm_last_error.restype = C.c_char_p
    L.cjm_version.restype = C.c_int
    _lib = L
    return L


def _check(status: int, where: str, ok=(0,)):
    if status not in ok:
        raise CJMError(status, where, lib().cjm_last_error().decode(errors="replace"))
    return status


# ------------------------------------------------------------ marshalling
def _dev_ptr(t, name):
    """(pointer, pitch in elements) of a 2-D fp64 CUDA tensor with unit column stride."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.dim() == 2
            and t.stride(1) == 1):
        raise TypeError(f"{name}: expected a 2-D float64 CUDA tensor with unit column stride")
    return C.c_void_p(t.data_ptr()), t.stride(0)


def _host_ptr(a, name):
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or a.ndim != 2 or a.strides[1] != 8:
            raise TypeError(f"{name}: expected a 2-D float64 array with unit column stride")
        return C.c_void_p(a.ctypes.data), a.strides[0] // 8
    import torch
    if isinstance(a, torch.Tensor) and not a.is_cuda and a.dtype == torch.float64 and a.dim() == 2 \
            and a.stride(1) == 1:
        return C.c_void_p(a.data_ptr()), a.stride(0)
    raise TypeError(f"{name}: expected a host float64 array")


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------ API
def cjm_default_options(**kw) -> Options:
    o = Options()
    lib().cjm_default_options(C.byref(o))
    for k, v in kw.items():
        if k == "nccl_id":
            continue
        setattr(o, k, v)
    return o


def cjm_schedule(stencil: int, nx: int, ny: int, tol: float, order: int = ORDER_LEBEDEV23) -> dict:
    kmin, kmax = C.c_double(), C.c_double()
    m, P = C.c_longlong(), C.c_longlong()
    _check(lib().cjm_schedule(stencil, nx, ny, tol, order, C.byref(kmin), C.byref(kmax),
                              C.byref(m), C.byref(P), None, None, 0), "cjm_schedule")
    t = np.empty(P.value, dtype=np.int64)
    w = np.empty(P.value, dtype=np.float64)
    _check(lib().cjm_schedule(stencil, nx, ny, tol, order, None, None, None, None,
                              t.ctypes.data_as(C.POINTER(C.c_longlong)),
                              w.ctypes.data_as(C.POINTER(C.c_double)), P.value), "cjm_schedule")
    return dict(kappa_min=kmin.value, kappa_max=kmax.value, m_min=m.value, P=P.value, t=t, w=w)


def cjm_slab(ny: int, world_size: int, rank: int) -> tuple[int, int]:
    y0, n = C.c_int(), C.c_int()
    _check(lib().cjm_slab(ny, world_size, rank, C.byref(y0), C.byref(n)), "cjm_slab")
    return y0.value, n.value


def cjm_halo_plan(ny: int, r: int, world_size: int, rank: int) -> list[dict]:
    """Halo messages of `rank`: dicts with peer, send_row, recv_row, rows
    (local buffer rows, ghost rows included)."""
    msgs = (HaloMsg * 2)()
    n = C.c_int()
    _check(lib().cjm_halo_plan(ny, r, world_size, rank, msgs, C.byref(n)), "cjm_halo_plan")
    return [dict(peer=m.peer, send_row=m.send_row, recv_row=m.recv_row, rows=m.rows)
            for m in msgs[:n.value]]


def cjm_buffer_layout(nx: int) -> tuple[int, int]:
    """(ld, col0) of the library's internal row layout for nx interior columns."""
    ld, c0 = C.c_longlong(), C.c_int()
    _check(lib().cjm_buffer_layout(nx, C.byref(ld), C.byref(c0)), "cjm_buffer_layout")
    return ld.value, c0.value


def cjm_halo_xfers(nx: int, ny: int, depth: int, world_size: int, rank: int) -> tuple[list[dict], int]:
    """The element-level transfers of the library's NCCL halo exchange
    (peer, send_off, recv_off, count in doubles of the internal layout) and ld."""
    xs = (HaloXfer * 2)()
    n, ld = C.c_int(), C.c_longlong()
    _check(lib().cjm_halo_xfers(nx, ny, depth, world_size, rank, xs, C.byref(n), C.byref(ld)),
           "cjm_halo_xfers")
    return [dict(peer=x.peer, send_off=x.send_off, recv_off=x.recv_off, count=x.count)
            for x in xs[:n.value]], ld.value


def cjm_get_nccl_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().cjm_get_nccl_id(buf), "cjm_get_nccl_id")
    return buf.raw


class Plan:
    """Owns a cjm_plan_t (cjm_plan ... cjm_plan_destroy)."""

    def __init__(self, stencil: int, nx: int, ny: int, h: float, tol: float,
                 bc: int = BC_DIRICHLET, nccl_id: bytes | None = None, **options):
        self._h = C.c_void_p()
        o = cjm_default_options(**options)
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = C.cast(self._id_buf, C.c_void_p)
        _check(lib().cjm_plan(C.byref(self._h), stencil, nx, ny, h, bc, tol, C.byref(o)), "cjm_plan")
        self.stencil, self.nx, self.ny, self.h, self.tol = stencil, nx, ny, h, tol
        self._load_info()

    def _load_info(self):
        info = self.info()
        self.reach, self.y0, self.ny_local = info["reach"], info["y0"], info["ny_local"]
        self.ghost_rows, self.rhs_ghost_rows = info["ghost_rows"], info["rhs_ghost_rows"]
        self.P = info["cycle_len"]

    def info(self) -> dict:
        rep, r, y0, nyl, w = Report(), C.c_int(), C.c_int(), C.c_int(), C.POINTER(C.c_double)()
        _check(lib().cjm_plan_info(self._h, C.byref(rep), C.byref(r), C.byref(y0), C.byref(nyl),
                                   C.byref(w)), "cjm_plan_info")
        d = rep.as_dict()
        d.update(reach=r.value, y0=y0.value, ny_local=nyl.value,
                 weights=np.ctypeslib.as_array(w, shape=(rep.cycle_len,)).copy())
        return d

    def _check_shapes(self, rhs, u):
        r, gu, gr = self.reach, self.ghost_rows, self.rhs_ghost_rows
        if tuple(u.shape) != (self.ny_local + 2 * gu, self.nx + 2 * r):
            raise ValueError(f"u: shape {tuple(u.shape)}, plan expects "
                             f"{(self.ny_local + 2 * gu, self.nx + 2 * r)}")
        if tuple(rhs.shape) != (self.ny_local + 2 * gr, self.nx):
            raise ValueError(f"rhs: shape {tuple(rhs.shape)}, plan expects "
                             f"{(self.ny_local + 2 * gr, self.nx)}")

    def solve(self, rhs, u, stream=None, ok=(0,)) -> dict:
        """cjm_solve on device tensors; u is updated in place."""
        self._check_shapes(rhs, u)
        rp, rl = _dev_ptr(rhs, "rhs")
        up, ul = _dev_ptr(u, "u")
        rep = Report()
        _check(lib().cjm_solve(self._h, rp, rl, up, ul, _stream(stream), C.byref(rep)), "cjm_solve", ok)
        return rep.as_dict()

    def solve_ref(self, rhs, u, u_ref, real_tol: float, stream=None, ok=(0,)) -> dict:
        """cjm_solve_ref: stop on max|u - u_ref| <= real_tol."""
        self._check_shapes(rhs, u)
        if tuple(u_ref.shape) != (self.ny_local, self.nx):
            raise ValueError("u_ref: interior shape (ny_local, nx) expected")
        rp, rl = _dev_ptr(rhs, "rhs")
        up, ul = _dev_ptr(u, "u")
        ep, el = _dev_ptr(u_ref, "u_ref")
        rep = Report()
        _check(lib().cjm_solve_ref(self._h, rp, rl, up, ul, ep, el, real_tol, _stream(stream),
                                   C.byref(rep)), "cjm_solve_ref", ok)
        return rep.as_dict()

    def solve_host(self, rhs, u, stream=None, ok=(0,)) -> dict:
        """cjm_solve_host on host arrays; u is updated in place."""
        self._check_shapes(rhs, u)
        rp, rl = _host_ptr(rhs, "rhs")
        up, ul = _host_ptr(u, "u")
        rep = Report()
        _check(lib().cjm_solve_host(self._h, rp, rl, up, ul, _stream(stream), C.byref(rep)),
               "cjm_solve_host", ok)
        return rep.as_dict()

    def sweeps(self, rhs, u, first: int, count: int, stream=None) -> dict:
        self._check_shapes(rhs, u)
        rp, rl = _dev_ptr(rhs, "rhs")
        up, ul = _dev_ptr(u, "u")
        rep = Report()
        _check(lib().cjm_sweeps(self._h, rp, rl, up, ul, first, count, _stream(stream), C.byref(rep)),
               "cjm_sweeps")
        return rep.as_dict()

    def residual(self, rhs, u, stream=None) -> tuple[float, float]:
        self._check_shapes(rhs, u)
        rp, rl = _dev_ptr(rhs, "rhs")
        up, ul = _dev_ptr(u, "u")
        l2, li = C.c_double(), C.c_double()
        _check(lib().cjm_residual(self._h, rp, rl, up, ul, _stream(stream), C.byref(l2), C.byref(li)),
               "cjm_residual")
        return l2.value, li.value

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().cjm_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


MASK_KEYS = ("W", "E", "S", "N", "C")


class MaskPlan(Plan):
    """Owns a generic 5-point mask plan (cjm_plan_mask ... cjm_plan_destroy).
    `mask` (optional): dict W, E, S, N, C of ny x nx float64 CUDA tensors,
    passed to cjm_mask_set."""

    def __init__(self, nx: int, ny: int, kappa_min: float, kappa_max: float, tol: float,
                 mask: dict | None = None, **options):
        self._h = C.c_void_p()
        self._id_buf = None
        o = cjm_default_options(**options)
        _check(lib().cjm_plan_mask(C.byref(self._h), nx, ny, kappa_min, kappa_max, tol, C.byref(o)),
               "cjm_plan_mask")
        self.stencil, self.nx, self.ny, self.h, self.tol = STENCIL_MASK, nx, ny, 1.0, tol
        self._load_info()
        if mask is not None:
            self.mask_set(mask)

    def mask_set(self, mask: dict, stream=None) -> None:
        ptrs, lds = [], set()
        for k in MASK_KEYS:
            t = mask[k]
            if tuple(t.shape) != (self.ny, self.nx):
                raise ValueError(f"mask[{k!r}]: shape {tuple(t.shape)}, plan expects {(self.ny, self.nx)}")
            p, ld = _dev_ptr(t, f"mask[{k!r}]")
            ptrs.append(p)
            lds.add(ld)
        if len(lds) != 1:
            raise ValueError("mask arrays must share one pitch")
        _check(lib().cjm_mask_set(self._h, *ptrs, lds.pop(), _stream(stream)), "cjm_mask_set")


class MaskPlanN(Plan):
    """Owns a generic (2m+1)^2 mask plan (cjm_plan_mask_n ... cjm_plan_destroy),
    m = radius 1 or 2.  `planes` (optional): list of (2m+1)^2 entries, each a
    ny x nx float64 CUDA tensor or None (absent neighbour), in mask order
    q = (dy+m)(2m+1) + (dx+m); passed to cjm_mask_set_n."""

    def __init__(self, nx: int, ny: int, radius: int, kappa_min: float, kappa_max: float,
                 tol: float, planes: list | None = None, **options):
        self._h = C.c_void_p()
        self._id_buf = None
        o = cjm_default_options(**options)
        _check(lib().cjm_plan_mask_n(C.byref(self._h), nx, ny, radius, kappa_min, kappa_max, tol,
                                     C.byref(o)), "cjm_plan_mask_n")
        self.stencil, self.nx, self.ny, self.h, self.tol = STENCIL_MASK, nx, ny, 1.0, tol
        self.radius = radius
        self._load_info()
        if planes is not None:
            self.mask_set(planes)

    def mask_set(self, planes: list, stream=None) -> None:
        q = (2 * self.radius + 1) ** 2
        if len(planes) != q:
            raise ValueError(f"a radius-{self.radius} mask has {q} planes, got {len(planes)}")
        ptrs, lds = [], set()
        for k, t in enumerate(planes):
            if t is None:
                ptrs.append(None)
                continue
            if tuple(t.shape) != (self.ny, self.nx):
                raise ValueError(f"planes[{k}]: shape {tuple(t.shape)}, plan expects {(self.ny, self.nx)}")
            p, ld = _dev_ptr(t, f"planes[{k}]")
            ptrs.append(p)
            lds.add(ld)
        if len(lds) != 1:
            raise ValueError("mask planes must share one pitch")
        arr = (C.c_void_p * q)(*ptrs)
        _check(lib().cjm_mask_set_n(self._h, arr, lds.pop(), _stream(stream)), "cjm_mask_set_n")


def cjm_plan_mask_n(nx, ny, radius, kappa_min, kappa_max, tol=1e-8, planes=None,
                    **options) -> MaskPlanN:
    return MaskPlanN(nx, ny, radius, kappa_min, kappa_max, tol, planes=planes, **options)


def cjm_plan_mask(nx, ny, kappa_min, kappa_max, tol=1e-8, mask=None, **options) -> MaskPlan:
    return MaskPlan(nx, ny, kappa_min, kappa_max, tol, mask=mask, **options)


def cjm_mask_set(plan: MaskPlan, mask: dict, stream=None) -> None:
    plan.mask_set(mask, stream)


def cjm_mask_bounds(mask: dict, iters: int = 0) -> tuple[float, float]:
    """Host estimate (kappa_min, kappa_max) of D^-1 A for a mask of host
    float64 arrays (cjm_mask_bounds: power iteration, bipartite symmetry)."""
    arrs = [np.ascontiguousarray(mask[k], dtype=np.float64) for k in MASK_KEYS]
    ny, nx = arrs[0].shape
    if any(a.shape != (ny, nx) for a in arrs):
        raise ValueError("mask arrays must share one shape")
    kmin, kmax = C.c_double(), C.c_double()
    _check(lib().cjm_mask_bounds(nx, ny, *[C.c_void_p(a.ctypes.data) for a in arrs], nx, iters,
                                 C.byref(kmin), C.byref(kmax)), "cjm_mask_bounds")
    return kmin.value, kmax.value


def cjm_mask_bounds_n(planes: list, iters: int = 0) -> tuple[float, float]:
    """Host estimate (kappa_min, kappa_max) of D^-1 A for a (2m+1)^2 mask of
    host float64 planes (None = absent), cjm_mask_bounds_n."""
    q = len(planes)
    m = {9: 1, 25: 2}.get(q)
    if m is None:
        raise ValueError("a square mask has 9 or 25 planes")
    arrs = [None if c is None else np.ascontiguousarray(c, dtype=np.float64) for c in planes]
    centre = arrs[m * (2 * m + 1) + m]
    if centre is None:
        raise ValueError("the centre plane c_C is required")
    if centre.ndim != 2:
        raise ValueError("planes must be 2-D (ny, nx) arrays")
    ny, nx = centre.shape
    for k, a in enumerate(arrs):
        if a is not None and a.shape != (ny, nx):
            raise ValueError(f"planes[{k}]: shape {a.shape}, centre plane is {(ny, nx)}")
    ptrs = (C.c_void_p * q)(*[None if a is None else a.ctypes.data for a in arrs])
    kmin, kmax = C.c_double(), C.c_double()
    _check(lib().cjm_mask_bounds_n(nx, ny, m, ptrs, nx, iters, C.byref(kmin), C.byref(kmax)),
           "cjm_mask_bounds_n")
    return kmin.value, kmax.value


def cjm_plan(stencil, nx, ny, h, bc=BC_DIRICHLET, tol=1e-8, **options) -> Plan:
    return Plan(stencil, nx, ny, h, tol, bc=bc, **options)


def cjm_plan_info(plan: Plan) -> dict:
    return plan.info()


def cjm_solve(plan: Plan, rhs, u, stream=None) -> dict:
    return plan.solve(rhs, u, stream)


def cjm_solve_ref(plan: Plan, rhs, u, u_ref, real_tol, stream=None) -> dict:
    return plan.solve_ref(rhs, u, u_ref, real_tol, stream)


def cjm_solve_host(plan: Plan, rhs, u, stream=None) -> dict:
    return plan.solve_host(rhs, u, stream)


def cjm_sweeps(plan: Plan, rhs, u, first, count, stream=None) -> dict:
    return plan.sweeps(rhs, u, first, count, stream)


def cjm_residual(plan: Plan, rhs, u, stream=None):
    return plan.residual(rhs, u, stream)


def cjm_plan_destroy(plan: Plan) -> None:
    plan.close()


def cjm_pool_trim() -> int:
    """Free the library's cached device buffers; returns the bytes released."""
    b = C.c_longlong()
    _check(lib().cjm_pool_trim(C.byref(b)), "cjm_pool_trim")
    return b.value


def cjm_version() -> int:
    return lib().cjm_version()
