"""Pins the oracle (oracle/d2q37_oracle.c) before it is trusted as the checker.

* Reference known answers: frozen t0 / weights and moment identities
  (proj/tests/test_model.cpp:87-142, acceptance.cpp C1-C2), delta impulse,
  rest population, permutation and periodicity (test_kernels.cpp:114-276).
* Reference outputs: tests/golden/*.npz, written by the unmodified reference
  (tests/golden/make_golden.py) -- bit-exact for propagate and halo_exchange,
  <= 1e-13 for collide and steps (the reference build contracts into FMA,
  the oracle does not).
* Published RNG answers: std::mt19937_64's 10000th output ([rand.predef]) and
  the Random123 Philox4x32-10 known-answer vectors.
* Builder-defined wall bc (no reference counterpart): reflection impulse,
  permutation (exact mass conservation), y-mirror symmetry.
"""
import numpy as np
import pytest

from conftest import golden, max_rel


def test_velocity_set_census_and_order(po):
    """acceptance C1, test_model.cpp:38-92."""
    m = po.orc_model()
    v = list(zip(m.cx.tolist(), m.cy.tolist()))
    assert len(set(v)) == 37
    census = {}
    for cx, cy in v:
        census[cx * cx + cy * cy] = census.get(cx * cx + cy * cy, 0) + 1
    assert census == {0: 1, 1: 4, 2: 4, 4: 4, 5: 8, 8: 4, 9: 4, 10: 8}
    keys = [(cx * cx + cy * cy, cx, cy) for cx, cy in v]
    assert keys == sorted(keys)
    for cx, cy in v:
        assert (-cx, -cy) in v and (cy, cx) in v and (-cx, cy) in v


def test_frozen_weights_and_t0(po):
    """test_model.cpp:87-117 (multiprecision values)."""
    m = po.orc_model()
    assert m.t0 == pytest.approx(0.69795332201968309, rel=1e-12)
    frozen = {(0, 0): 0.23315066913235250, (1, 0): 0.10730609154221900, (1, 1): 0.05766785988879488,
              (2, 0): 0.01420821615845075, (2, 1): 0.00535304900051378, (2, 2): 0.00101193759267358,
              (3, 0): 0.00024530102775772, (3, 1): 0.00028341425299420}
    for (cx, cy), w in frozen.items():
        i = int(np.nonzero((m.cx == cx) & (m.cy == cy))[0][0])
        assert m.w[i] == pytest.approx(w, rel=1e-10)
    assert np.all(m.w > 0)
    assert abs(m.w.sum() - 1.0) < 1e-14


def test_moment_conditions(po):
    """test_model.cpp:119-142 / acceptance C2."""
    m = po.orc_model()
    t0 = m.t0
    t2, t3, t4 = t0 * t0, t0 ** 3, t0 ** 4

    def mom(a, b):
        acc = 0.0
        for i in range(37):
            term = m.w[i]
            for _ in range(a):
                term *= m.cx[i]
            for _ in range(b):
                term *= m.cy[i]
            acc += term
        return acc

    for a, b, want in [(0, 0, 1.0), (2, 0, t0), (4, 0, 3 * t2), (2, 2, t2), (6, 0, 15 * t3), (4, 2, 3 * t3),
                       (8, 0, 105 * t4), (6, 2, 15 * t4), (4, 4, 9 * t4)]:
        assert abs(mom(a, b) - want) < 1e-12
    assert abs(mom(1, 0)) < 1e-15 and abs(mom(3, 0)) < 1e-15 and abs(mom(1, 2)) < 1e-15


def test_model_matches_reference_golden(po):
    """Oracle constants vs the reference build: t0 and the Hermite table exact, weights within 16 ulp."""
    g = golden("ref_model.npz")
    m = po.orc_model()
    assert np.array_equal(m.cx, g["cx"]) and np.array_equal(m.cy, g["cy"])
    assert m.t0 == float(g["t0"])
    assert np.max(np.abs(m.w.view(np.int64) - g["w"].view(np.int64))) <= 16
    assert max_rel(m.eq[m.eq != 0], g["eq"][m.eq != 0]) < 1e-14


def test_mt19937_64_known_answer(po):
    """C++ [rand.predef]: the 10000th output of a default-seeded mt19937_64 is 9981545732273789042."""
    u = po.mt64_u01(5489, 10000)
    assert u[-1] == float(9981545732273789042 >> 11) * 2.0 ** -53


def test_philox_known_answers(po):
    """Random123 kat_vectors for philox4x32-10."""
    assert po.philox([0, 0, 0, 0], [0, 0]) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert po.philox([0xffffffff] * 4, [0xffffffff] * 2) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert po.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]) == \
        [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


@pytest.mark.parametrize("name", ["ref_random_16x32.npz", "ref_random_5x12.npz"])
def test_oracle_vs_reference_golden(po, name):
    g = golden(name)
    lx, ly, vl = int(g["lx"]), int(g["ly"]), int(g["vl_csoa"])
    init = g["init"]
    # generator: same mt19937_64 stream, equilibrium within FMA rounding
    assert max_rel(po.orc_lattice("random", lx, ly, seed=int(g["seed"])), init) < 1e-14
    # propagate + halo_exchange: bit-exact (pure data movement)
    assert np.array_equal(po.orc_propagate(init), g["propagate_soa"])
    assert np.array_equal(po.orc_propagate(init), g["propagate_csoa"])
    assert np.array_equal(po.orc_halo_fill(po.orc_to_padded(init, 1), lx, ly, 1), g["padded_soa"])
    assert np.array_equal(po.orc_halo_fill(po.orc_to_padded(init, vl), lx, ly, vl), g["padded_csoa"])
    # collide / steps: FMA vs no-FMA rounding only
    out, bad = po.orc_collide(init, float(g["omega_collide"]))
    assert not bad
    assert max_rel(out, g["collide"]) < 1e-13
    assert max_rel(out, g["oracle_collide"]) < 1e-13
    st, _ = po.orc_step(init, float(g["omega_step"]), int(g["steps"]))
    assert max_rel(st, g["step"]) < 1e-12


def test_oracle_vs_live_reference(po):
    """Same checks against the compiled reference when oracle/_ref is present."""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    lx, ly = 16, 32
    init = po.ref_random_lattice(lx, ly, 31)
    assert np.array_equal(po.orc_propagate(init), po.ref_oracle_propagate(init))
    for layout, vl in ((po.SOA, 1), (po.CSOA, 2), (po.CSOA, 8)):
        s = po.RefSim(layout, lx, ly, vl, workers=2)
        s.load(init)
        s.halo_exchange()
        assert np.array_equal(s.raw(), po.orc_halo_fill(po.orc_to_padded(init, vl), lx, ly, vl))
    assert max_rel(po.orc_collide(init, 1.7)[0], po.ref_oracle_collide(init, 1.7)) < 1e-13


@pytest.mark.parametrize("vl", [1, 2, 4, 8])
@pytest.mark.parametrize("bc", [0, 1])
def test_padded_restatement_consistent(po, vl, bc):
    """halo fill + padded propagate (kernels.cpp path) == canonical pull (validation.cpp path)."""
    lx, ly = 9, 48
    init = po.orc_lattice("random", lx, ly, seed=3)
    buf = po.orc_halo_fill(po.orc_to_padded(init, vl), lx, ly, vl, bc)
    out = po.orc_from_padded(po.orc_propagate_padded(buf, lx, ly, vl), lx, ly, vl)
    assert np.array_equal(out, po.orc_propagate(init, bc))


def test_delta_impulse_and_rest_population(po):
    """test_kernels.cpp:114-146."""
    m = po.orc_model()
    p10 = int(np.nonzero((m.cx == 1) & (m.cy == 0))[0][0])
    a = np.zeros((37, 8, 8))
    a[p10, 3, 5] = 1.0
    out = po.orc_propagate(a)
    want = np.zeros_like(a)
    want[p10, 4, 5] = 1.0
    assert np.array_equal(out, want)
    init = po.orc_lattice("random", 6, 16, seed=7)
    assert np.array_equal(po.orc_propagate(init)[0], init[0])


def test_permutation_and_periodicity(po):
    """test_kernels.cpp:240-276."""
    init = po.orc_lattice("random", 4, 8, seed=77)
    a = init
    for _ in range(4 * 8):
        a = po.orc_propagate(a)
    assert np.array_equal(a, init)
    out = po.orc_propagate(init)
    for p in range(37):
        assert np.array_equal(np.sort(out[p].ravel()), np.sort(init[p].ravel()))


def test_wall_known_answers(po):
    """Builder wall KATs: reflection impulse, exact permutation, y-mirror symmetry."""
    m = po.orc_model()
    ybar = m.ymirror()
    p7 = int(np.nonzero((m.cx == 1) & (m.cy == -1))[0][0])
    a = np.zeros((37, 8, 16))
    a[p7, 3, 0] = 1.0
    out = po.orc_propagate(a, po.BC_WALL)
    want = np.zeros_like(a)
    want[ybar[p7], 4, 0] = 1.0
    assert np.array_equal(out, want)
    # pure permutation of all values: mass conserved bit for bit
    init = po.orc_lattice("random", 12, 20, seed=5)
    out = po.orc_propagate(init, po.BC_WALL)
    assert np.array_equal(np.sort(out.ravel()), np.sort(init.ravel()))
    # a y-mirror-symmetric state stays symmetric through wall steps
    sym = 0.5 * (init + init[ybar][:, :, ::-1])
    st, _ = po.orc_step(sym, 0.8, 3, po.BC_WALL)
    mirrored = st[ybar][:, :, ::-1]
    assert max_rel(st, mirrored) < 1e-13


def test_rt_init_shape(po):
    """Config-0 init: hot below the interface, cold above, uniform pressure, at rest."""
    from conftest import macros_fields
    a = po.orc_lattice("rt", 32, 64, seed=12345)
    rho, ux, uy, temp = macros_fields(po, a)
    assert np.all(np.abs(temp[:, :20] - 1.5) < 2e-3) and np.all(np.abs(temp[:, 44:] - 0.5) < 2e-3)
    assert np.max(np.abs(rho * temp - 1.0)) < 1e-12
    assert np.max(np.abs(ux)) < 1e-12 and np.max(np.abs(uy)) < 1e-12


def test_oracle_collide_conservation(po):
    """test_model.cpp:282-306: mass, momentum, energy conserved by collide_site."""
    rng = np.random.default_rng(42)
    m = po.orc_model()
    for _ in range(100):
        f = 0.01 + 0.99 * rng.random(37)
        omega = 0.1 + 1.8 * rng.random()
        out, bad = po.orc_collide_site(f, omega)
        assert not bad
        d = out - f
        assert abs(d.sum()) / f.sum() < 1e-11
        assert abs((m.cx * d).sum()) < 1e-11 and abs((m.cy * d).sum()) < 1e-11
        e = ((m.cx ** 2 + m.cy ** 2) * f).sum()
        assert abs(((m.cx ** 2 + m.cy ** 2) * d).sum()) / e < 1e-11


def test_oracle_nonphysical(po):
    _, bad = po.orc_collide_site(-np.ones(37), 1.0)
    assert bad
