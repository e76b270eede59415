"""Long-run parity of the bench step (FUSED2) against the unmodified reference and the oracle.

BASELINE north_star: the full multi-step run must agree with the reference CPU implementation within
1e-12 (max relative error) after one step and 1e-9 after 100 steps, on the populations and on the
derived density, velocity and temperature (model.cpp:242-257).  The reference's own long-run check
is acceptance C4 (acceptance.cpp:141-169: 100 steps of lbm::step) and its validation driver steps the
oracle the same way (validation.cpp:84-90).  Here:

* the periodic cases run against the UNMODIFIED reference (oracle/_ref, `lbm::step` through its
  LatticeState / ThreadPool, built with the reference's FMA contraction);
* the wall cases run against the C oracle (the reference has no wall bc), on a lattice
  large enough (4096 x 2048) to take the split launch whose interior form the bench times.

Velocity is compared relative to the largest speed of the reference field (u is ~0 in most of the RT
state, so an elementwise relative error of u is not meaningful); density and temperature elementwise.
"""
import os

import numpy as np
import pytest

from conftest import macros_fields, max_rel

pytestmark = pytest.mark.gpu

OMEGA = 0.8


def _fields_close(po, got, want, tol):
    rg, uxg, uyg, tg = macros_fields(po, got)
    rw, uxw, uyw, tw = macros_fields(po, want)
    speed = max(float(np.max(np.abs(uxw))), float(np.max(np.abs(uyw))))
    errs = {"f": max_rel(got, want), "rho": max_rel(rg, rw), "T": max_rel(tg, tw),
            "u": max(float(np.max(np.abs(uxg - uxw))), float(np.max(np.abs(uyg - uyw)))) / speed}
    assert all(v <= tol for v in errs.values()), errs
    return errs


def _ref_steps(po, init, n):
    lx, ly = init.shape[1], init.shape[2]
    r = po.RefSim(po.AOS, lx, ly, 1, workers=os.cpu_count() or 1)
    r.load(init)
    r.step(OMEGA, n)
    return r.dump()


@pytest.mark.parametrize("layout", ["soa", "banded"])
def test_fused2_one_and_two_steps_vs_unmodified_reference(gpu, lbm, po, layout):
    """Config-0 recipe (256 x 1024 RT), periodic, omega 0.8: one step (the odd step: FUSED on SoA, a
    one-step sweep on the banded store) and two steps (one FUSED2 sweep) within 1e-12 of the
    unmodified reference's lbm::step, populations and derived fields."""
    lx, ly = 256, 1024
    init = lbm.make_lattice("rt", lx, ly, seed=12345)
    for n in (1, 2):
        s = lbm.Simulation(layout, lx, ly, 1, device=0, bc="periodic", variant="fused2")
        s.load(init)
        s.step(OMEGA, n)
        _fields_close(po, s.dump(), _ref_steps(po, init, n), 1e-12)
        s.close()


@pytest.mark.parametrize("layout", ["soa", "banded"])
def test_fused2_100_steps_vs_unmodified_reference(gpu, lbm, po, layout):
    """acceptance.cpp:141-169 at the BASELINE tolerance: 100 steps as 50 FUSED2 sweeps (config-0 RT
    recipe, periodic, omega 0.8) against 100 steps of the unmodified reference: <= 1e-9 on the
    populations, rho, u and T."""
    lx, ly = 256, 1024
    init = lbm.make_lattice("rt", lx, ly, seed=12345)
    s = lbm.Simulation(layout, lx, ly, 1, device=0, bc="periodic", variant="fused2")
    s.load(init)
    s.step(OMEGA, 100)
    assert s.time_step == 100
    _fields_close(po, s.dump(), _ref_steps(po, init, 100), 1e-9)


_ORACLE_200: dict = {}


@pytest.mark.slow
@pytest.mark.parametrize("layout", ["soa", "banded"])
def test_fused2_200_steps_walls_split_path_vs_oracle(gpu, lbm, po, layout):
    """validation.cpp:84-90 (the oracle stepped alongside) at the bench step's own code path: a
    4096 x 2048 RT lattice with walls -- past the small-lattice threshold, so SoA runs the
    bench's sweep kernel (k_step2_pair, one launch per sweep with the wall images in the ghost rows) -- 200
    steps (100 sweeps) within 1e-9 of the C oracle on populations and derived fields; after one sweep
    within 1e-12."""
    lx, ly = 4096, 2048
    init = lbm.make_lattice("rt", lx, ly, seed=2024)
    s = lbm.Simulation(layout, lx, ly, 1, device=0, bc="wall", variant="fused2")
    s.load(init)
    s.step(OMEGA, 2)
    if not _ORACLE_200:  # the oracle's 200 steps are the test's cost: stepped once for both stores
        want2, bad2 = po.orc_step(init, OMEGA, 2, po.BC_WALL)
        want, bad = po.orc_step(want2, OMEGA, 198, po.BC_WALL)
        _ORACLE_200.update(want2=want2, want=want, bad=bad2 or bad)
    assert not _ORACLE_200["bad"]
    _fields_close(po, s.dump(), _ORACLE_200["want2"], 1e-12)
    s.step(OMEGA, 198)
    _fields_close(po, s.dump(), _ORACLE_200["want"], 1e-9)
    if layout == "banded":  # the last user: drop the 2 x 2.5 GB of cached oracle states
        _ORACLE_200.clear()
