"""Multi-rank (row-slab) decomposition on CPU with the gloo backend.

SURVEY section 8(e), rows a9 (halo exchange every sweep) and a10 (residual
allreduce per check).  Each rank owns the slab cjm_slab() gives it, exchanges
halos exactly as cjm_halo_plan() (the library's own host logic, the same
function its NCCL exchange uses) lays them out, sweeps its slab with the
oracle and allreduces (sum, max) of the per-slab reduction.  The gathered
field must be bitwise equal to the single-domain oracle, and the allreduced
norms must match the single-domain ones.

test_library_transfer_list_deep_halos runs the library's K-fused multi-GPU
schedule itself with gloo as the transport: host buffers in the library's
internal layout (cjm_buffer_layout), the exact transfers its NCCL exchange
issues (cjm_halo_xfers: peers, element offsets, counts; the g rows once per
solve, the u rows after every K-sweep launch), H = K r deep halos.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1705_00103_b200 import cjm, inputs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, stencil, nx, ny, nsweeps, check_every, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = oracle.reach(stencil)
        u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=11)
        s = oracle.schedule(stencil, nx, ny, 1e-8)
        g_all = oracle.rhs_to_g(stencil, h, b)
        y0, nyl = cjm.cjm_slab(ny, world, rank)
        # local slab of the padded field: global rows y0-r .. y0+nyl+r
        u = u0[y0:y0 + nyl + 2 * r].copy()
        g = g_all[y0:y0 + nyl].copy()
        msgs = cjm.cjm_halo_plan(ny, r, world, rank)
        norms = []
        for k in range(nsweeps):
            if k % check_every == 0:
                ss, mm = oracle.delta_norms(stencil, u, g)
                t = torch.tensor([ss], dtype=torch.float64)
                m = torch.tensor([mm], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
                dist.all_reduce(m, op=dist.ReduceOp.MAX)
                norms.append((t.item(), m.item()))
            u = oracle.sweep(stencil, u, g, s["w"][k % s["P"]])
            # halo exchange (row a9): post every receive / send of this sweep
            reqs, bufs = [], []
            for msg in msgs:
                send = torch.from_numpy(np.ascontiguousarray(u[msg["send_row"]:msg["send_row"] + msg["rows"]]))
                recv = torch.empty_like(send)
                reqs.append(dist.isend(send, msg["peer"]))
                reqs.append(dist.irecv(recv, msg["peer"]))
                bufs.append((msg, recv))
            for q in reqs:
                q.wait()
            for msg, recv in bufs:
                u[msg["recv_row"]:msg["recv_row"] + msg["rows"]] = recv.numpy()
        gathered = [None] * world
        dist.all_gather_object(gathered, (y0, nyl, u[r:r + nyl].copy()))
        if rank == 0:
            out.put((gathered, norms))
    finally:
        dist.destroy_process_group()


def _run(world, stencil, nx, ny, nsweeps, check_every):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, world, port, stencil, nx, ny, nsweeps,
                                               check_every, q)) for rk in range(world)]
    for p in procs:
        p.start()
    gathered, norms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return gathered, norms


@pytest.mark.parametrize("world,stencil,nx,ny", [(2, 9, 37, 50), (2, 17, 23, 41), (3, 5, 30, 29)])
def test_row_slabs_match_single_domain(world, stencil, nx, ny):
    nsweeps, check_every = 12, 5
    gathered, norms = _run(world, stencil, nx, ny, nsweeps, check_every)
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=11)
    s = oracle.schedule(stencil, nx, ny, 1e-8)
    g = oracle.rhs_to_g(stencil, h, b)
    u = u0
    ref_norms = []
    for k in range(nsweeps):
        if k % check_every == 0:
            ref_norms.append(oracle.delta_norms(stencil, u, g))
        u = oracle.sweep(stencil, u, g, s["w"][k % s["P"]])
    field = np.concatenate([blk for _, _, blk in sorted(gathered, key=lambda t: t[0])])
    assert field.shape == (ny, nx + 2 * r)
    assert np.array_equal(field, u[r:r + ny])           # bitwise, ghosts columns included
    for (ss, mm), (rs, rm) in zip(norms, ref_norms):
        assert ss == pytest.approx(rs, rel=1e-13)       # different summation order
        assert mm == rm                                 # max is order-free


def test_halo_plan_geometry():
    for ny, world, r in [(100, 4, 1), (101, 3, 2), (4096 * 8, 8, 1)]:
        for rank in range(world):
            y0, nyl = cjm.cjm_slab(ny, world, rank)
            msgs = cjm.cjm_halo_plan(ny, r, world, rank)
            peers = [m["peer"] for m in msgs]
            assert peers == [p for p in (rank - 1, rank + 1) if 0 <= p < world]
            for m in msgs:
                assert m["rows"] == r
                if m["peer"] == rank - 1:
                    assert m["send_row"] == r and m["recv_row"] == 0
                else:
                    assert m["send_row"] == nyl and m["recv_row"] == nyl + r
                # what I send to a peer lands on the peer's ghost rows that
                # mirror the same global rows
                py0, pnyl = cjm.cjm_slab(ny, world, m["peer"])
                pm = [x for x in cjm.cjm_halo_plan(ny, r, world, m["peer"]) if x["peer"] == rank][0]
                assert y0 + m["send_row"] - r == py0 + pm["recv_row"] - r
    with pytest.raises(cjm.CJMError):
        cjm.cjm_halo_plan(8, 2, 4, 0)    # slabs of 2 rows < 2r+1


# ----------------------------------------------------------------------------
# The library's own transfer list on gloo: deep halos of K-fused launches
# ----------------------------------------------------------------------------

def _xfer_worker(rank, world, port, stencil, nx, ny, K, nlaunch, out):
    """One rank of the K-fused multi-GPU schedule, with the device buffers
    replaced by flat host buffers in the library's internal layout
    (cjm_buffer_layout) and the NCCL exchange replaced by gloo send / recv of
    exactly the transfers the library issues (cjm_halo_xfers: peer, element
    offsets, counts).  The K sweeps of a launch are the oracle's sweeps on the
    slab extended by its H = K r ghost rows (the rows inside the global grid
    computed redundantly, as the kernel does)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r = oracle.reach(stencil)
        H = K * r
        u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=19)
        s = oracle.schedule(stencil, nx, ny, 1e-8)
        g_all = oracle.rhs_to_g(stencil, h, b)
        y0, nyl = cjm.cjm_slab(ny, world, rank)
        ld, c0 = cjm.cjm_buffer_layout(nx)
        xs, ld2 = cjm.cjm_halo_xfers(nx, ny, H, world, rank)
        assert ld2 == ld
        rows = nyl + 2 * H
        ubuf = np.zeros(rows * ld)
        gbuf = np.zeros(rows * ld)
        U, G = ubuf.reshape(rows, ld), gbuf.reshape(rows, ld)
        cols = slice(c0 - r, c0 + nx + r)
        # global row y (ghost rows -r..-1 and ny..ny+r-1) <-> u0 row y + r
        lo_g, hi_g = max(-r, y0 - H), min(ny + r, y0 + nyl + H)   # rows that exist globally
        for y in range(lo_g, hi_g):
            U[y - y0 + H, cols] = u0[y + r]
        for y in range(y0, y0 + nyl):                            # g: my interior rows only
            G[y - y0 + H, c0:c0 + nx] = g_all[y]

        def exchange(buf):
            reqs, recvs = [], []
            for x in xs:
                send = torch.from_numpy(buf[x["send_off"]:x["send_off"] + x["count"]].copy())
                recv = torch.empty(x["count"], dtype=torch.float64)
                reqs += [dist.isend(send, x["peer"]), dist.irecv(recv, x["peer"])]
                recvs.append((x, recv))
            for q in reqs:
                q.wait()
            for x, recv in recvs:
                buf[x["recv_off"]:x["recv_off"] + x["count"]] = recv.numpy()

        exchange(gbuf)                    # once per solve: the neighbours' g rows
        exchange(ubuf)                    # u_0's halo
        a, e = lo_g - y0 + H, hi_g - y0 + H   # local rows of the extended slab
        norms = []
        for k in range(nlaunch):
            ext = U[a:e, cols].copy()     # outermost r rows act as fixed ghosts
            gext = G[a + r:e - r, c0:c0 + nx]
            if k == 0:
                ss, mm = oracle.delta_norms(stencil, U[H - r:H + nyl + r, cols],
                                            G[H:H + nyl, c0:c0 + nx])
                t = torch.tensor([ss, mm], dtype=torch.float64)
                dist.all_reduce(t[:1], op=dist.ReduceOp.SUM)
                dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
                norms.append((t[0].item(), t[1].item()))
            for l in range(K):
                ext = oracle.sweep(stencil, ext, gext, s["w"][(k * K + l) % s["P"]])
            U[H:H + nyl, cols] = ext[H - a:H - a + nyl]
            exchange(ubuf)
        gathered = [None] * world
        dist.all_gather_object(gathered, (y0, U[H:H + nyl, cols].copy()))
        if rank == 0:
            out.put((gathered, norms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,stencil,nx,ny,K", [(2, 9, 37, 50, 4), (3, 17, 23, 61, 3),
                                                   (2, 5, 30, 29, 2), (4, 9, 19, 60, 1)])
def test_library_transfer_list_deep_halos(world, stencil, nx, ny, K):
    nlaunch = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xfer_worker, args=(rk, world, port, stencil, nx, ny, K, nlaunch, q))
             for rk in range(world)]
    for p in procs:
        p.start()
    gathered, norms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r = oracle.reach(stencil)
    u0, b, h = inputs.test_problem(nx, ny, r, init="random", seed=19)
    s = oracle.schedule(stencil, nx, ny, 1e-8)
    g = oracle.rhs_to_g(stencil, h, b)
    ss, mm = oracle.delta_norms(stencil, u0, g)
    assert norms[0][0] == pytest.approx(ss, rel=1e-13) and norms[0][1] == mm
    want = oracle.sweeps(stencil, u0, g, s["w"], 0, nlaunch * K)
    field = np.concatenate([blk for _, blk in sorted(gathered, key=lambda t: t[0])])
    assert np.array_equal(field, want[r:r + ny])
