"""CPU-side checks of the product library (no GPU needed).

* the C-ABI library loads and exports every symbol include/d2q37_b200.h declares;
* the product's host model (VelocityModel::d2q37 restatement) and initialisers
  agree with the oracle bit for bit and with the reference's frozen values;
* argument validation mirrors the reference's std::invalid_argument cases
  (layout.cpp:14-23) and fails before any device work;
* metric formulas reproduce the reference's Table-1 cross-checks
  (acceptance.cpp:202-212, test_metrics.cpp:13-39);
* the C++ host header include/lbm_b200/lbm_b200.hpp compiles against the C-ABI.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "d2q37_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(d2q37_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lbm):
    lib = ctypes.CDLL(lbm.library_path())
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a(lbm):
    out = subprocess.run(["cuobjdump", "--list-elf", lbm.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_model_equals_oracle_model(lbm, po):
    m, o = lbm.model(), po.orc_model()
    assert np.array_equal(m.velocities[:, 0], o.cx) and np.array_equal(m.velocities[:, 1], o.cy)
    assert np.array_equal(m.weights, o.w)
    assert m.t0 == o.t0
    assert np.array_equal(m.eq_table, o.eq)


def test_product_model_frozen_values(lbm):
    m = lbm.model()
    assert m.t0 == pytest.approx(0.69795332201968309, rel=1e-12)
    assert m.weights[0] == pytest.approx(0.23315066913235250, rel=1e-10)
    assert abs(m.weights.sum() - 1.0) < 1e-14
    g = golden("ref_model.npz")
    assert m.t0 == float(g["t0"])


def test_reference_table_is_sign_symmetric(lbm):
    """The FAST kernels use one Hermite row per (+-a, +-b) quadruple; the reference's table qualifies."""
    g = golden("ref_model.npz")
    cx, cy, eq = g["cx"], g["cy"], g["eq"]
    xodd = np.array([1, 0, 0, 1, 0, 1, 0, 1, 0, 0, 1, 0, 1, 0])
    yodd = np.array([0, 1, 0, 1, 0, 0, 1, 0, 1, 0, 1, 0, 1, 0])
    for i in range(37):
        for j in range(37):
            if abs(cx[j]) == abs(cx[i]) and abs(cy[j]) == abs(cy[i]):
                sx = np.where((xodd == 1) & (np.sign(cx[i]) != np.sign(cx[j])), -1.0, 1.0)
                sy = np.where((yodd == 1) & (np.sign(cy[i]) != np.sign(cy[j])), -1.0, 1.0)
                assert np.array_equal(eq[j], eq[i] * sx * sy), (i, j)


@pytest.mark.parametrize("kind", ["random", "rt", "c2", "philox"])
def test_initialisers_equal_oracle(lbm, po, kind):
    a = lbm.make_lattice(kind, 12, 40, seed=99)
    b = po.orc_lattice(kind, 12, 40, seed=99)
    assert np.array_equal(a, b)


def test_initialisers_param_kinds(lbm, po):
    m = lbm.model()
    a = lbm.make_lattice("equilibrium", 6, 8, params=[1.1, 0.02, -0.01, m.t0])
    assert np.array_equal(a, po.orc_lattice("equilibrium", 6, 8, mac=[1.1, 0.02, -0.01, m.t0]))
    a = lbm.make_lattice("shear", 6, 8, params=[0.02, m.t0])
    assert np.array_equal(a, po.orc_lattice("shear", 6, 8, amp=0.02, temp=m.t0))


def test_random_lattice_matches_reference_generator(lbm, po):
    """Same mt19937_64 stream as make_random_lattice (lattice.cpp:8-23); FMA-only differences."""
    g = golden("ref_random_16x32.npz")
    a = lbm.make_lattice("random", 16, 32, seed=int(g["seed"]))
    assert float(np.max(np.abs(a - g["init"]) / g["init"])) < 1e-14


def test_host_model_helpers(lbm):
    """module.cpp:135-170 helpers (test_smoke.py:44-71 analogue)."""
    m = lbm.model()
    feq = m.equilibrium(1.2, 0.05, -0.03, m.t0 * 1.1)
    rho, ux, uy, temp = m.macros(feq)
    assert abs(rho - 1.2) < 1e-12 and abs(ux - 0.05) < 1e-12 and abs(uy + 0.03) < 1e-12
    assert abs(temp - m.t0 * 1.1) < 1e-12
    f = np.random.default_rng(3).uniform(0.01, 1.0, 37)
    out = m.collide_site(f, 1.4)
    assert abs(out.sum() - f.sum()) / f.sum() < 1e-12
    with pytest.raises(lbm.NonPhysicalError):
        m.macros(-np.ones(37))


@pytest.mark.parametrize("args,msg", [
    (("caosoa", 8, 16, 3), "power of two"),
    (("caosoa", 8, 18, 4), "divisible"),
    (("csoa", 8, 16, 3), "power of two"),
    (("csoa", 8, 18, 4), "divisible"),
    (("csoa", 8, 16, 8), "shorter than its halo"),
    (("soa", 0, 16, 1), "positive"),
    (("hex", 8, 16, 1), "unknown layout"),
])
def test_geometry_validation_like_reference(lbm, args, msg):
    """layout.cpp:14-23 error cases, raised as ValueError (std::invalid_argument) before device work."""
    with pytest.raises(ValueError, match=msg):
        lbm.Simulation(*args)


def test_bad_initialiser_arguments(lbm):
    with pytest.raises(ValueError):
        lbm.make_lattice("equilibrium", 4, 4)  # needs params
    with pytest.raises(ValueError):
        lbm.make_lattice("random", 4, 4, out=np.empty((37, 4, 5)))


def test_metric_formulas_reproduce_table1(lbm):
    """acceptance.cpp:202-212 / test_metrics.cpp:13-39."""
    assert lbm.propagate_gbps(1024, 8192, 37, 0.0125, "nt") == pytest.approx(398.0, rel=0.01)
    assert lbm.collide_gflops(1024, 8192, 6600.0, 0.0503) == pytest.approx(1100.0, rel=0.01)
    assert lbm.mlups(1024, 8192, 0.0503) == pytest.approx(166.0, rel=0.01)
    assert lbm.mlups(4608, 12288, 0.55025) == pytest.approx(103.0, rel=0.01)
    assert lbm.propagate_gbps(256, 512, 37, 0.001, "rfo") == pytest.approx(
        1.5 * lbm.propagate_gbps(256, 512, 37, 0.001, "nt"), rel=1e-15)
    with pytest.raises(ValueError):
        lbm.mlups(4, 4, 0.0)


def test_halo_plan(lbm):
    """26 pop-rows per face (15 + 8 + 3), the minimal set read by a pull from |cy| <= 3."""
    lo, hi = lbm.halo_plan()
    m = lbm.model()
    assert len(lo) == len(hi) == 26
    for d, p in lo:
        assert m.velocities[p, 1] <= -d
    for d, p in hi:
        assert m.velocities[p, 1] >= d
    assert sum(1 for d, _ in hi if d == 1) == 15 and sum(1 for d, _ in hi if d == 2) == 8


def test_slab_neighbours(lbm):
    assert [lbm.slab_neighbors(r, 4, "wall") for r in range(4)] == [(-1, 1), (0, 2), (1, 3), (2, -1)]
    assert [lbm.slab_neighbors(r, 4, "periodic") for r in range(4)] == [(3, 1), (0, 2), (1, 3), (2, 0)]
    assert lbm.slab_neighbors(0, 1, "periodic") == (-1, -1)


def test_cpp_header_compiles(lbm, tmp_path):
    """include/lbm_b200/lbm_b200.hpp (the reference-shaped C++ API) builds and links against the C-ABI."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "lbm_b200/lbm_b200.hpp"
#include <cstdio>
int main() {
    using namespace lbm_b200;
    const VelocityModel& m = VelocityModel::d2q37();
    CanonicalLattice c = make_random_lattice(4, 8, 1);
    if (c.values.size() != 37u * 4 * 8 || !(m.t0() > 0.69 && m.t0() < 0.70)) return 1;
    try { LatticeState s(LayoutKind::CSoA, Geometry{8, 18, 3, 3, 4}); return 2; }
    catch (const std::invalid_argument&) {}
    std::printf("%.17g\n", m.t0());
    return mlups(1024, 8192, 0.0503) > 166.0 ? 0 : 3;
}
''')
    exe = tmp_path / "t"
    libdir = os.path.dirname(lbm.library_path())
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{os.path.join(ROOT, 'include')}", str(src), "-o", str(exe),
                    f"-L{libdir}", "-ld2q37_b200", f"-Wl,-rpath,{libdir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert float(r.stdout) == lbm.model().t0


def test_validation_first_divergence_order_and_defaults(lbm):
    """first_divergence scans x, then y, then p (validation.cpp:59-70); the options default to
    the reference's ValidationOptions (validation.hpp:44-58)."""
    from paper_1804_01918_b200 import validation as v

    want = np.zeros((37, 3, 4))
    got = want.copy()
    assert v.first_divergence(got, want) is None
    got[5, 2, 0] = 1.0
    got[30, 1, 3] = 2.0
    got[2, 1, 3] = -0.0  # a sign bit differs: bitwise compare catches it
    d = v.first_divergence(got, want)
    assert (d.x, d.y, d.p, d.got, d.want) == (1, 3, 2, -0.0, 0.0)
    o = v.ValidationOptions()
    assert o.geometries == [(16, 32), (64, 128)] and o.vls == [1, 2, 4, 8]
    assert o.layouts == ["aos", "soa", "csoa", "caosoa"] and (o.steps, o.omega, o.seed) == (10, 1.0, 12345)
    assert o.corrupt_population == -1


def test_product_quadrature_satisfies_the_moment_conditions(lbm):
    """The shipped quadrature table (csrc/d2q37_host.cpp) solves the conditions model.cpp:101-181
    derives it from: lattice moments sum_i w_i cx^a cy^b equal the 2-D Gaussian's of variance t0 for
    (a, b) in {(0,0) (2,0) (4,0) (2,2) (6,0) (4,2) (6,2) (4,4) (8,0)} (test_model.cpp:119-142), all
    weights positive, one weight per shell."""
    m = lbm.model()
    cx, cy = m.velocities[:, 0].astype(float), m.velocities[:, 1].astype(float)
    w, t0 = m.weights, m.t0

    def gauss(k):
        return 0.0 if k % 2 else float(np.prod(np.arange(k - 1, 0, -2, dtype=float))) * t0 ** (k // 2)

    for a, b in ((0, 0), (2, 0), (4, 0), (2, 2), (6, 0), (4, 2), (6, 2), (4, 4), (8, 0)):
        lat = float(np.sum(w * cx ** a * cy ** b))
        assert abs(lat - gauss(a) * gauss(b)) <= 1e-12 * max(1.0, abs(gauss(a) * gauss(b))), (a, b)
    assert np.all(w > 0)
    n2 = cx * cx + cy * cy
    for s in np.unique(n2):
        assert len(np.unique(w[n2 == s])) == 1
