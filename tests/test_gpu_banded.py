"""The band-blocked device store (layout "banded", csrc/d2q37_banded.cu): the FUSED2 bench store.

Every case compares through the C-ABI library with the SoA / CAoSoA single-sweep step
(k_collide<FAST, SHIFT>, itself pinned to the oracle and the reference in
test_gpu_parity.py) bit for bit: a two-step sweep of the banded store must be exactly two
FUSED steps, a one-step sweep one, whatever the faces, the band edges and the slab cut --
the analogue of the reference's layout / worker invariance (test_kernels.cpp:361-397).
"""
import numpy as np
import pytest

from conftest import macros_fields, max_rel

pytestmark = pytest.mark.gpu


def sim(lbm, layout, lx, ly, vl=1, **kw):
    return lbm.Simulation(layout, lx, ly, vl, device=0, **kw)


def fused_ref(lbm, init, omega, n, bc):
    lx, ly = init.shape[1], init.shape[2]
    r = sim(lbm, "soa", lx, ly, bc=bc, variant="fused")
    r.load(init)
    r.step(omega, n)
    out = r.dump()
    r.close()
    return out


def test_load_dump_round_trip_bitwise(gpu, lbm):
    """LatticeState::load / dump (lattice.hpp:18-19) through the banded store: the canonical
    array comes back bit for bit (owner slots; halo copies are written alongside)."""
    for lx, ly in ((5, 12), (3, 121), (17, 360), (8, 245)):
        init = lbm.make_lattice("random", lx, ly, seed=lx * 1000 + ly)
        s = sim(lbm, "banded", lx, ly)
        s.load(init)
        assert np.array_equal(s.dump(), init)
        assert np.array_equal(s.dump(which=1), np.zeros_like(init))  # zeroed at creation (layout.cpp:101)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
@pytest.mark.parametrize("lx,ly", [(64, 128), (37, 300), (130, 245), (5, 12), (1, 16), (9, 13), (300, 123),
                                   (6, 121), (4, 241), (3, 125), (2, 126)])
def test_banded_fused2_bitwise_equals_fused(gpu, lbm, bc, lx, ly):
    """Two-step sweeps of the banded store == single fused steps bit for bit: band edges (ly = 2*120 + 1
    leaves a 1-row last band, 121 / 125 / 126 put the last band's rows inside the previous band's high
    halo), degenerate x (lx = 1, 2, 3 wrap more than once), odd step counts (one-step sweeps) and both
    y faces."""
    init = lbm.make_lattice("random", lx, ly, seed=17 + ly)
    s = sim(lbm, "banded", lx, ly, bc=bc, variant="fused2")
    s.load(init)
    r = sim(lbm, "soa", lx, ly, bc=bc, variant="fused")
    r.load(init)
    for n in (2, 1, 4, 3):
        s.step(1.3, n)
        r.step(1.3, n)
        assert np.array_equal(s.dump(), r.dump()), n
    assert s.time_step == r.time_step == 10


def test_banded_bc_change_between_calls(gpu, lbm):
    """The halo slots hold every periodic image whatever the step's faces, so a wall run followed by a
    periodic run (and back) equals the same sequence of fused steps."""
    lx, ly = 24, 250
    init = lbm.make_lattice("random", lx, ly, seed=5)
    s = sim(lbm, "banded", lx, ly, variant="fused2")
    r = sim(lbm, "soa", lx, ly, variant="fused")
    s.load(init)
    r.load(init)
    for bc, n in (("wall", 4), ("periodic", 3), ("wall", 2), ("periodic", 6)):
        s.step(1.1, n, bc=bc)
        r.step(1.1, n, bc=bc)
        assert np.array_equal(s.dump(), r.dump()), bc


def test_banded_graph_replay_bitwise(gpu, lbm):
    """step(n >= 40) replays captured graphs of ten sweeps: equal to single fused steps."""
    lx, ly = 64, 256
    init = lbm.make_lattice("random", lx, ly, seed=4)
    a = sim(lbm, "banded", lx, ly, variant="fused2", bc="wall")
    a.load(init)
    a.step(1.1, 47)
    assert np.array_equal(a.dump(), fused_ref(lbm, init, 1.1, 47, "wall"))


def test_banded_vs_oracle_config0(gpu, lbm, po):
    """Config 0 recipe (256 x 1024 RT, walls, omega 0.8): 2 steps within 1e-12 of the oracle on the
    populations and on rho, u, T (model.cpp:242-257)."""
    lx, ly = 256, 1024
    init = lbm.make_lattice("rt", lx, ly, seed=12345)
    s = sim(lbm, "banded", lx, ly, bc="wall", variant="fused2")
    s.load(init)
    s.step(0.8, 2)
    got = s.dump()
    want, bad = po.orc_step(init, 0.8, 2, po.BC_WALL)
    assert not bad
    assert max_rel(got, want) <= 1e-12
    for a, b in zip(macros_fields(po, got), macros_fields(po, want)):
        assert max_rel(a, b) <= 1e-12 or float(np.max(np.abs(a - b))) <= 1e-12 * float(np.max(np.abs(b)))


def test_banded_device_rt_init_equals_soa(gpu, lbm):
    """init_rt_device on the banded store writes the same per-site values as on SoA."""
    lx, ly = 96, 700
    a = sim(lbm, "banded", lx, ly)
    a.init_rt_device(77)
    b = sim(lbm, "soa", lx, ly)
    b.init_rt_device(77)
    assert np.array_equal(a.dump(), b.dump())


def test_banded_moments_and_conservation(gpu, lbm):
    """Global mass / momentum / energy (acceptance.cpp:141-169) on the banded store: equal to the SoA
    store's sums, and conserved to 1e-11 over 20 periodic steps."""
    lx, ly = 64, 512
    init = lbm.make_lattice("random", lx, ly, seed=9)
    a = sim(lbm, "banded", lx, ly, variant="fused2")
    a.load(init)
    b = sim(lbm, "soa", lx, ly)
    b.load(init)
    m0 = a.moments()
    assert np.allclose(m0, b.moments(), rtol=1e-14, atol=1e-12)
    a.step(1.2, 20)
    m1 = a.moments()
    assert abs(m1[0] - m0[0]) <= 1e-11 * abs(m0[0])
    assert abs(m1[3] - m0[3]) <= 1e-11 * abs(m0[3])


def test_banded_nonphysical_raises(gpu, lbm):
    """NonPhysicalError (model.hpp:28-30) from a banded sweep."""
    lx, ly = 16, 130
    bad = lbm.make_lattice("random", lx, ly, seed=3)
    bad[:, 5, 125] = -1.0
    s = sim(lbm, "banded", lx, ly, variant="fused2")
    s.load(bad)
    with pytest.raises(lbm.NonPhysicalError):
        s.step(1.0, 2)


def test_banded_unsupported_verbs_fail_loudly(gpu, lbm):
    """The padded-buffer verbs, UNFUSED steps and STRICT math have no banded form: an error, never a
    silent fallback."""
    s = sim(lbm, "banded", 8, 24)
    s.load(lbm.make_lattice("random", 8, 24, seed=1))
    for call in (lambda: s.bc("periodic"), lambda: s.propagate_only(), lambda: s.collide(1.0),
                 lambda: s.read_padded(), lambda: s.step(1.0, 1, variant="unfused")):
        with pytest.raises((ValueError, RuntimeError, NotImplementedError)):
            call()
    with pytest.raises(ValueError):
        sim(lbm, "banded", 8, 11)  # ly >= 12


def test_banded_convert_and_lbdump(gpu, lbm, tmp_path):
    """convert (layout.cpp:105-116) to and from the banded store, and LBDUMP01 files (dump.cpp:44-70):
    bit for bit."""
    lx, ly = 33, 250
    init = lbm.make_lattice("random", lx, ly, seed=11)
    a = sim(lbm, "soa", lx, ly)
    a.load(init)
    b = lbm.convert(a, "banded")
    assert np.array_equal(b.dump(), init)
    c = lbm.convert(b, "aos")
    assert np.array_equal(c.dump(), init)
    path = str(tmp_path / "b.lbdump")
    b.save_dump(path)
    d = sim(lbm, "banded", lx, ly)
    d.load_dump(path)
    assert np.array_equal(d.dump(), init)
    e = sim(lbm, "soa", lx, ly)
    e.load_dump(path)
    assert np.array_equal(e.dump(), init)


@pytest.mark.parametrize("nslabs", [2, 3])
@pytest.mark.parametrize("bc", ["periodic", "wall"])
@pytest.mark.parametrize("lx,ly", [(32, 252), (7, 72), (130, 726)])
def test_banded_slab_group_bitwise_equals_single_domain(gpu, lbm, nslabs, bc, lx, ly):
    """Banded y-slabs (6-row halos of 37 populations per face and sweep, written into the halo slots)
    are bit for bit the single domain: 2 and 3 slabs on one GPU, slabs of 24 rows to multi-band slabs,
    odd step counts (one-step sweeps after the exchange)."""
    init = lbm.make_lattice("random", lx, ly, seed=41)
    ref = sim(lbm, "soa", lx, ly, bc=bc, variant="fused")
    ref.load(init)
    grp = lbm.SlabGroup("banded", lx, ly, 1, nslabs, bc=bc, variant="fused2")
    grp.load(init)
    for n in (2, 3, 4):
        ref.step(1.1, n)
        grp.step(1.1, n)
        assert np.array_equal(grp.dump(), ref.dump()), n


def test_banded_nccl_self_ring_bitwise_equals_single_domain(gpu, lbm):
    """Banded FUSED2 through the real NCCL transport: a 1-rank ring whose 6-row halos go through
    ncclSend/ncclRecv to self before every sweep (and before the odd one-step sweep)."""
    import torch  # noqa: F401  (torch's libnccl.so.2 is the one the library binds to)

    lx, ly = 32, 256
    init = lbm.make_lattice("random", lx, ly, seed=47)
    s = lbm.Simulation.slab("banded", lx, ly, 1, rank=0, nranks=1, nccl_id=lbm.nccl_unique_id(),
                            variant="fused2")
    s.load(init)
    s.step(1.2, 7)
    assert np.array_equal(s.dump(), fused_ref(lbm, init, 1.2, 7, "periodic"))


@pytest.mark.slow
def test_banded_full_size_bitwise(gpu, lbm):
    """The bench workload (4096 x 16384 RT, walls, omega 0.8) on the banded store: 4 steps as two
    sweeps equal 4 single fused steps of the CAoSoA32 store bit for bit."""
    lx, ly = 4096, 16384
    s = sim(lbm, "banded", lx, ly, bc="wall", variant="fused2")
    s.init_rt_device(4242)
    s.step(0.8, 4)
    got = s.dump()
    s.close()
    r = sim(lbm, "caosoa", lx, ly, 32, bc="wall", variant="fused")
    r.init_rt_device(4242)
    r.step(0.8, 4)
    want = r.dump()
    r.close()
    assert np.array_equal(got, want)
