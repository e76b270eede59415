"""The streamed run (d2q37_run_canonical / Simulation.run): load + step + dump as one call.

The reference's host-side sequence is LatticeState::load, n x lbm::step, LatticeState::dump
(lattice.hpp:18-19, kernels.cpp:276-283; module.cpp:44-99 for the Python Simulation).  The streamed
run must return exactly what those three verbs return, bit for bit, whether it pipelines the copies
under the sweeps (single SoA wall domain, FUSED2, even n: y-chunks swept as parallelograms of
sweeps) or falls back to the three verbs one after another (every other case).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OMEGA = 0.8


class _Env:
    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _three_verbs(lbm, init, n, bc="wall", variant="fused2"):
    lx, ly = init.shape[1:]
    s = lbm.Simulation("soa", lx, ly, device=0, bc=bc, variant=variant)
    s.load(init)
    s.step(OMEGA, n)
    out = s.dump()
    s.close()
    return out


@pytest.mark.parametrize("rows,first,last,n", [(480, 240, 120, 20), (240, 120, 240, 100), (600, 600, 600, 2),
                                               (2040, 480, 240, 40), (720, 120, 6, 12), (24, 8, 8, 8)])
def test_streamed_run_bitwise_equals_load_step_dump(gpu, lbm, rows, first, last, n):
    """Several chunk heights, including chunks shorter than the rows-per-sweep skew accumulates to
    (240 rows against 50 sweeps x 8 rows), chunks of a few rows and a single sweep."""
    lx, ly = (1024, 2400) if rows > 24 else (256, 600)
    init = lbm.make_lattice("rt", lx, ly, seed=777)
    want = _three_verbs(lbm, init, n)
    s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    with _Env(D2Q37_STREAM_ROWS=rows, D2Q37_STREAM_FIRST=first, D2Q37_STREAM_LAST=last):
        got = s.run(init, OMEGA, n)
    assert np.array_equal(got, want)
    assert s.time_step == n and s.last_run_mode == "pipelined_walls"
    # the lattice is left in the state the three verbs leave it in: stepping on agrees too
    s.step(OMEGA, 3)
    assert np.array_equal(s.dump(), _three_verbs(lbm, init, n + 3))
    s.close()


@pytest.mark.parametrize("skew", [6, 8, 14])
def test_streamed_run_in_place_and_repeated(gpu, lbm, skew):
    """out may be the input array; a second run on the same handle starts from the new input.  Any
    rows-per-sweep skew >= 6 gives the same result."""
    lx, ly = 512, 1920
    init = lbm.make_lattice("rt", lx, ly, seed=5)
    s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    buf = init.copy()
    with _Env(D2Q37_STREAM_ROWS=360, D2Q37_STREAM_FIRST=120, D2Q37_STREAM_SKEW=skew):
        s.run(buf, OMEGA, 10, out=buf)
        assert np.array_equal(buf, _three_verbs(lbm, init, 10))
        s.run(buf, OMEGA, 6, out=buf)  # an odd sweep count: the state ends in the other buffer
    assert np.array_equal(buf, _three_verbs(lbm, init, 16))
    assert np.array_equal(s.dump(), buf)
    s.close()


@pytest.mark.parametrize("lx,ly,n", [(64, 1201, 10), (8, 700, 6), (3, 486, 4), (1000, 481, 2), (200, 1000, 30)])
def test_streamed_run_odd_extents(gpu, lbm, lx, ly, n):
    """Odd and non-band-multiple heights (the last chunk ends at ly whatever its parity), very narrow
    lattices, default chunk heights."""
    init = lbm.make_lattice("rt", lx, ly, seed=lx + ly)
    s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    got = s.run(init, OMEGA, n)
    assert np.array_equal(got, _three_verbs(lbm, init, n))
    with _Env(D2Q37_STREAM_ROWS=124, D2Q37_STREAM_FIRST=36, D2Q37_STREAM_LAST=12):
        got = s.run(init, OMEGA, n)
    assert np.array_equal(got, _three_verbs(lbm, init, n))
    s.close()


def test_streamed_run_default_chunks_larger_lattice(gpu, lbm):
    """Default chunk heights (2 bands doubling up to 37-band chunks, halving to 1 band at the top wall) on
    a lattice wide enough for the lockstep plan's even split (4096 columns on 148 CTAs)."""
    lx, ly = 4096, 4800
    a = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    a.init_rt_device(2018)
    init = a.dump()
    a.step(OMEGA, 8)
    want = a.dump()
    got = a.run(init, OMEGA, 8)
    assert np.array_equal(got, want)
    a.close()


@pytest.mark.parametrize("lx,ly,n,rows", [(512, 2400, 20, 0), (512, 2400, 100, 240), (64, 1203, 6, 36),
                                          (4096, 2560, 8, 0), (256, 1124, 2, 0)])
def test_streamed_run_periodic_bitwise(gpu, lbm, lx, ly, n, rows):
    """y-periodic domains (the reference's own boundary mode, kernels.cpp:197-234): the two pieces at the
    seam are swept first, with the periodic images between their sweeps, then the wave of chunks."""
    init = lbm.make_lattice("rt", lx, ly, seed=ly)
    want = _three_verbs(lbm, init, n, bc="periodic")
    s = lbm.Simulation("soa", lx, ly, device=0, bc="periodic", variant="fused2")
    env = dict(D2Q37_STREAM_ROWS=rows, D2Q37_STREAM_FIRST=max(12, rows // 4), D2Q37_STREAM_LAST=12) if rows else {}
    buf = init.copy()
    with _Env(**env):
        s.run(buf, OMEGA, n, out=buf)
    assert np.array_equal(buf, want) and s.last_run_mode == "pipelined_periodic"
    s.step(OMEGA, 2)  # the periodic images left in the ghost rows are the final state's
    assert np.array_equal(s.dump(), _three_verbs(lbm, init, n + 2, bc="periodic"))
    s.close()


def test_streamed_run_periodic_vs_unmodified_reference(gpu, lbm, po):
    """load -> 4 x lbm::step -> dump of the unmodified reference (lattice.hpp:18-19, kernels.cpp:276-283)
    against one streamed run: populations within 1e-12."""
    lx, ly, n = 96, 1200, 4
    init = lbm.make_lattice("random", lx, ly, seed=31)
    ref = po.RefSim(po.AOS, lx, ly, 1, workers=os.cpu_count() or 1)
    ref.load(init)
    ref.step(OMEGA, n)
    s = lbm.Simulation("soa", lx, ly, device=0, bc="periodic", variant="fused2")
    got = s.run(init, OMEGA, n)
    want = ref.dump()
    assert s.last_run_mode == "pipelined_periodic"
    assert float(np.max(np.abs(got - want) / np.abs(want))) <= 1e-12
    s.close()


@pytest.mark.parametrize("bc,variant,n", [("periodic", "fused2", 6), ("wall", "fused2", 5), ("wall", "fused", 4),
                                          ("wall", "unfused", 2)])
def test_run_falls_back_to_three_verbs(gpu, lbm, bc, variant, n):
    lx, ly = 256, 600
    init = lbm.make_lattice("rt", lx, ly, seed=11)
    s = lbm.Simulation("soa", lx, ly, device=0, bc=bc, variant=variant)
    got = s.run(init, OMEGA, n)
    assert np.array_equal(got, _three_verbs(lbm, init, n, bc, variant)) and s.last_run_mode == "three_verbs"
    s.close()


def test_run_other_layouts_and_switch(gpu, lbm):
    """Layouts without the streamed path, and D2Q37_STREAM_RUN=0 on one that has it."""
    lx, ly = 256, 640
    init = lbm.make_lattice("rt", lx, ly, seed=3)
    want = _three_verbs(lbm, init, 4)
    for layout, vl in (("caosoa", 32), ("csoa", 8), ("aos", 1)):
        s = lbm.Simulation(layout, lx, ly, vl, device=0, bc="wall", variant="fused2")
        assert np.array_equal(s.run(init, OMEGA, 4), want)
        s.close()
    s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    with _Env(D2Q37_STREAM_RUN=0):
        assert np.array_equal(s.run(init, OMEGA, 4), want)
    s.close()


def test_streamed_run_reports_nonphysical(gpu, lbm):
    """A non-positive density inside a streamed sweep surfaces as NonPhysicalError from run()."""
    lx, ly = 512, 1200
    init = lbm.make_lattice("rt", lx, ly, seed=9)
    init[:, 100, 700] = -1.0
    s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
    with pytest.raises(lbm.NonPhysicalError):
        s.run(init, OMEGA, 4)
    s.close()
