"""bench.py's multi-rank host logic on CPU (gloo, world_size 2): the P2P transport set-up
(create -> blob all_gather -> connect) and its collective fallback to NCCL when any rank
cannot use peer memory -- every rank must take the same branch, and none may hang."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _FakeSim:
    def __init__(self, rank, transport):
        self.rank, self.transport, self.connected, self.closed = rank, transport, None, False

    def p2p_blob(self):
        return b"blob%d" % self.rank

    def p2p_connect(self, lo, hi):
        self.connected = (lo, hi)

    def close(self):
        self.closed = True


class _FakeLbm:
    def __init__(self, fail_rank, nccl=True):
        self.fail_rank = fail_rank
        self.nccl = nccl

    def nccl_unique_id(self):
        if not self.nccl:
            raise OSError("libnccl.so.2 not found")
        return b"id"

    @property
    def Simulation(self):
        outer = self

        class S:
            @staticmethod
            def slab(layout, lx, ly, vl, *, device, rank, nranks, bc, variant, transport="nccl", nccl_id=None):
                if transport == "p2p" and rank == outer.fail_rank:
                    raise ValueError("no peer memory here")
                return _FakeSim(rank, transport)
        return S


def _worker(rank, world, port, fail_rank, q, variant="fused", nccl=True):
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), BENCH_DIST_BACKEND="gloo")
    import argparse

    import bench

    d = bench.Dist()
    try:
        layout, vl = ("soa", 1) if variant == "fused2" else ("caosoa", 32)
        args = argparse.Namespace(transport="p2p", layout=layout, vl=vl, variant=variant)
        sim, transport = bench.make_slab(_FakeLbm(fail_rank, nccl), args, d, 0, 4096)
        q.put((rank, transport, sim.transport, sim.connected, args.variant, args.layout))
    finally:
        d.close()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_make_slab_transport_choice_is_collective(fail_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fail_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if fail_rank < 0:
        assert [got[r][0] for r in (0, 1)] == ["p2p", "p2p"]
        assert got[0][2] == (b"blob1", b"blob1") and got[1][2] == (b"blob0", b"blob0")
    else:
        assert [got[r][0] for r in (0, 1)] == ["nccl", "nccl"]
        assert [got[r][1] for r in (0, 1)] == ["nccl", "nccl"]


def test_make_slab_fused2_uses_nccl_on_every_rank():
    """FUSED2 slabs exchange 6-row halos through NCCL: no rank tries the peer-memory transport."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, -1, q, "fused2")) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [got[r][0] for r in (0, 1)] == ["nccl", "nccl"]
    assert [got[r][1] for r in (0, 1)] == ["nccl", "nccl"]


def test_make_slab_fused2_without_nccl_falls_back_to_p2p_on_every_rank():
    """NCCL missing (rank 0 cannot make an id): every rank learns it from the broadcast and takes the
    single-sweep CAoSoA32 P2P path -- none waits on a communicator that will not come."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, -1, q, "fused2", False)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, rest) for r, *rest in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [got[r][0] for r in (0, 1)] == ["p2p", "p2p"]
    assert [(got[r][3], got[r][4]) for r in (0, 1)] == [("fused", "caosoa")] * 2
