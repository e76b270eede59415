"""Multi-rank y-slab decomposition on CPU (gloo, world_size 2 and 3).

Runs the product's slab host logic -- the halo message plan
(d2q37_halo_plan: 26 pop-rows per face) and the neighbour map
(d2q37_slab_neighbors), issued in the same order as the NCCL exchange in
d2q37_nccl.cpp -- with torch.distributed/gloo moving the halos between
processes and the oracle doing the per-slab arithmetic.  Ghost entries that
are not in the plan are NaN, so a missing halo value would poison the result.
The decomposed run must equal the single-domain oracle bit for bit
(decomposition must not change any arithmetic).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slab_step(rank, nranks, slab, bc, omega, lbm, po):
    import torch

    m = po.orc_model()
    ybar = m.ymirror()
    lo_plan, hi_plan = lbm.halo_plan()
    lo_peer, hi_peer = lbm.slab_neighbors(rank, nranks, bc)
    npop, lx, n = slab.shape
    # pack (k_pack): send_lo <- rows d-1 of (d,p) in lo_plan; send_hi <- rows n-d of hi_plan
    send_lo = np.stack([slab[p, :, d - 1] for d, p in lo_plan])
    send_hi = np.stack([slab[p, :, n - d] for d, p in hi_plan])
    recv_lo = np.zeros_like(send_hi)
    recv_hi = np.zeros_like(send_lo)
    # exchange in the NCCL issue order: send hi, recv lo, send lo, recv hi
    t_rlo, t_rhi = torch.from_numpy(recv_lo), torch.from_numpy(recv_hi)
    reqs = []
    if hi_peer >= 0:
        reqs.append(dist.isend(torch.from_numpy(send_hi), hi_peer, tag=1))
    if lo_peer >= 0:
        reqs.append(dist.irecv(t_rlo, lo_peer, tag=1))
    if lo_peer >= 0:
        reqs.append(dist.isend(torch.from_numpy(send_lo), lo_peer, tag=2))
    if hi_peer >= 0:
        reqs.append(dist.irecv(t_rhi, hi_peer, tag=2))
    for r in reqs:
        r.wait()
    # padded slab: 3 ghost rows each side, unsent entries stay NaN
    P = np.full((npop, lx, n + 6), np.nan)
    P[:, :, 3:n + 3] = slab
    if lo_peer >= 0:
        for i, (d, p) in enumerate(hi_plan):  # our low ghosts come from the peer's send_hi
            P[p, :, 3 - d] = recv_lo[i]
    else:  # wall: ghost(-d, p) = f(d-1, ybar p)
        for d in (1, 2, 3):
            for p in range(npop):
                P[p, :, 3 - d] = slab[ybar[p], :, d - 1]
    if hi_peer >= 0:
        for i, (d, p) in enumerate(lo_plan):
            P[p, :, n + 2 + d] = recv_hi[i]
    else:
        for d in (1, 2, 3):
            for p in range(npop):
                P[p, :, n + 2 + d] = slab[ybar[p], :, n - d]
    # pull propagate on the padded slab, x periodic
    out = np.empty_like(slab)
    for p in range(npop):
        cx, cy = int(m.cx[p]), int(m.cy[p])
        out[p] = np.roll(P[p], cx, axis=0)[:, 3 - cy:3 - cy + n]
    assert not np.isnan(out).any(), "a ghost value outside the halo plan was read"
    new, bad = po.orc_collide(out, omega, nthreads=1)
    assert not bad
    return new


def _worker(rank, nranks, port, bc, steps, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import paper_1804_01918_b200 as lbm
    from oracle import pyoracle as po

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=nranks)
    try:
        lx, ly = 8, 12 * nranks
        glob = po.orc_lattice("random", lx, ly, seed=404)
        n = ly // nranks
        slab = np.ascontiguousarray(glob[:, :, rank * n:(rank + 1) * n])
        for _ in range(steps):
            slab = _slab_step(rank, nranks, slab, bc, 0.9, lbm, po)
        result_q.put((rank, slab))
    finally:
        dist.destroy_process_group()


def _exchange_faces(rank, nranks, slab, bc, lbm):
    """The y-major / P2P message: the 3 face rows of all 37 populations each way.  Returns the
    (lo, hi) ghost rows (3 each, lo ordered y = -3..-1, hi ordered y = n..n+2) or None at a wall."""
    import torch

    lo_peer, hi_peer = lbm.slab_neighbors(rank, nranks, bc)
    n = slab.shape[2]
    send_lo = np.ascontiguousarray(slab[:, :, 0:3])      # -> lo neighbour's high ghost rows
    send_hi = np.ascontiguousarray(slab[:, :, n - 3:n])  # -> hi neighbour's low ghost rows
    recv_lo, recv_hi = np.full_like(send_hi, np.nan), np.full_like(send_lo, np.nan)
    t_lo, t_hi = torch.from_numpy(recv_lo), torch.from_numpy(recv_hi)
    reqs = []
    if hi_peer >= 0:
        reqs.append(dist.isend(torch.from_numpy(send_hi), hi_peer, tag=3))
    if lo_peer >= 0:
        reqs.append(dist.irecv(t_lo, lo_peer, tag=3))
    if lo_peer >= 0:
        reqs.append(dist.isend(torch.from_numpy(send_lo), lo_peer, tag=4))
    if hi_peer >= 0:
        reqs.append(dist.irecv(t_hi, hi_peer, tag=4))
    for r in reqs:
        r.wait()
    return (recv_lo if lo_peer >= 0 else None), (recv_hi if hi_peer >= 0 else None)


def _push_step(slab, ghosts, bc, omega, po):
    """One step of a slab whose ghost rows were pushed by the neighbours after their previous
    step (the P2P schedule: compute, then push the new face rows)."""
    m = po.orc_model()
    ybar = m.ymirror()
    npop, lx, n = slab.shape
    P = np.full((npop, lx, n + 6), np.nan)
    P[:, :, 3:n + 3] = slab
    lo, hi = ghosts
    if lo is not None:
        P[:, :, 0:3] = lo
    else:
        for d in (1, 2, 3):
            for p in range(npop):
                P[p, :, 3 - d] = slab[ybar[p], :, d - 1]
    if hi is not None:
        P[:, :, n + 3:n + 6] = hi
    else:
        for d in (1, 2, 3):
            for p in range(npop):
                P[p, :, n + 2 + d] = slab[ybar[p], :, n - d]
    out = np.empty_like(slab)
    for p in range(npop):
        cx, cy = int(m.cx[p]), int(m.cy[p])
        out[p] = np.roll(P[p], cx, axis=0)[:, 3 - cy:3 - cy + n]
    assert not np.isnan(out).any()
    new, bad = po.orc_collide(out, omega, nthreads=1)
    assert not bad
    return new


def _push_worker(rank, nranks, port, bc, steps, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import paper_1804_01918_b200 as lbm
    from oracle import pyoracle as po

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=nranks)
    try:
        lx, ly = 8, 12 * nranks
        glob = po.orc_lattice("random", lx, ly, seed=405)
        n = ly // nranks
        slab = np.ascontiguousarray(glob[:, :, rank * n:(rank + 1) * n])
        ghosts = _exchange_faces(rank, nranks, slab, bc, lbm)  # prime after the load
        for _ in range(steps):
            slab = _push_step(slab, ghosts, bc, 0.9, po)
            ghosts = _exchange_faces(rank, nranks, slab, bc, lbm)  # push the new faces
        result_q.put((rank, slab))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_push_schedule_bitwise(nranks, bc, po):
    """The P2P / y-major schedule over real process boundaries: prime after load, then every
    step computes and pushes its 3 face rows (all 37 populations) into the neighbours' ghost
    rows for the next step; walls on the outer faces.  Bit-identical to one domain."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_push_worker, args=(r, nranks, port, bc, 3, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(nranks))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    result = np.concatenate([got[r] for r in range(nranks)], axis=2)
    want, bad = po.orc_step(po.orc_lattice("random", 8, 12 * nranks, seed=405), 0.9, 3,
                            po.BC_WALL if bc == "wall" else po.BC_PERIODIC)
    assert not bad
    assert np.array_equal(result, want)


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_slab_decomposition_bitwise(nranks, bc, po):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, nranks, port, bc, 3, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(nranks))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    result = np.concatenate([got[r] for r in range(nranks)], axis=2)
    lx, ly = 8, 12 * nranks
    want, bad = po.orc_step(po.orc_lattice("random", lx, ly, seed=404), 0.9, 3,
                            po.BC_WALL if bc == "wall" else po.BC_PERIODIC)
    assert not bad
    assert np.array_equal(result, want)


# --------------------------------------------------------------------------- FUSED2: 6-row halos per two steps

def _two_step_slab(rank, nranks, slab, omega, lbm, po):
    """One FUSED2 sweep of a periodic y-slab: rows 0..5 / n-6..n-1 of all 37 populations go to the
    lo / hi neighbour (k_pack6 -> NCCL -> k_unpack6 order), step 1 runs on rows -3 .. n+2 of the
    extended slab (pulls reach rows -6 .. n+5), step 2 on rows 0 .. n-1 from step 1's rows."""
    import torch

    m = po.orc_model()
    lo_peer, hi_peer = lbm.slab_neighbors(rank, nranks, "periodic")
    npop, lx, n = slab.shape
    h = 6
    send_lo = np.ascontiguousarray(slab[:, :, :h])
    send_hi = np.ascontiguousarray(slab[:, :, n - h:])
    recv_lo, recv_hi = np.full_like(send_hi, np.nan), np.full_like(send_lo, np.nan)
    t_rlo, t_rhi = torch.from_numpy(recv_lo), torch.from_numpy(recv_hi)
    reqs = [dist.isend(torch.from_numpy(send_hi), hi_peer, tag=1), dist.irecv(t_rlo, lo_peer, tag=1),
            dist.isend(torch.from_numpy(send_lo), lo_peer, tag=2), dist.irecv(t_rhi, hi_peer, tag=2)]
    for r in reqs:
        r.wait()
    ext = np.concatenate([recv_lo, slab, recv_hi], axis=2)  # rows -6 .. n+5

    def step(src, first, count):  # pull rows first .. first+count-1 of src (row 0 of src = y -6 or -3), collide
        out = np.empty((npop, lx, count))
        for p in range(npop):
            cx, cy = int(m.cx[p]), int(m.cy[p])
            out[p] = np.roll(src[p], cx, axis=0)[:, first - cy:first - cy + count]
        assert not np.isnan(out).any(), "a row outside the 6-row halo was read"
        new, bad = po.orc_collide(np.ascontiguousarray(out), omega, nthreads=1)
        assert not bad
        return new

    s1 = step(ext, 3, n + 6)  # y -3 .. n+2 (ext row index = y + 6)
    return step(s1, 3, n)  # y 0 .. n-1 (s1 row index = y + 3)


def _two_step_worker(rank, nranks, port, sweeps, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import paper_1804_01918_b200 as lbm
    from oracle import pyoracle as po

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=nranks)
    try:
        lx, ly = 8, 12 * nranks
        glob = po.orc_lattice("random", lx, ly, seed=406)
        n = ly // nranks
        slab = np.ascontiguousarray(glob[:, :, rank * n:(rank + 1) * n])
        for _ in range(sweeps):
            slab = _two_step_slab(rank, nranks, slab, 0.9, lbm, po)
        result_q.put((rank, slab))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 3])
def test_fused2_six_row_halo_schedule_bitwise(nranks, po):
    """The FUSED2 slab plan over real process boundaries: 6 rows x 37 populations per face per two
    steps are all a slab needs (unsent rows are NaN); 2 sweeps == 4 single-domain oracle steps."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_two_step_worker, args=(r, nranks, port, 2, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(nranks))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    result = np.concatenate([got[r] for r in range(nranks)], axis=2)
    want, bad = po.orc_step(po.orc_lattice("random", 8, 12 * nranks, seed=406), 0.9, 4, po.BC_PERIODIC)
    assert not bad
    assert np.array_equal(result, want)
