"""ctypes view of the oracle libraries -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` leg import this module.  It loads

* ``oracle/_build/liborc.so`` -- the plain-C restatement (d2q37_oracle.c), and
* ``oracle/_ref/liblbmref.so`` -- the unmodified reference compiled by
  oracle/Makefile, driven through ref_shim.cpp.

Arrays are numpy float64 in the reference's canonical order
``(p*lx + x)*ly + y`` (proj/include/lbm/dump.hpp:19-21), i.e. shape (37, lx, ly).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "liblbmref.so")
NPOP = 37
NMOM = 14
BC_PERIODIC, BC_WALL = 0, 1
AOS, SOA, CSOA, CAOSOA = 0, 1, 2, 3

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OrcModel(C.Structure):
    _fields_ = [
        ("cx", C.c_int * NPOP),
        ("cy", C.c_int * NPOP),
        ("shell", C.c_int * NPOP),
        ("w", C.c_double * NPOP),
        ("shell_w", C.c_double * 8),
        ("t0", C.c_double),
        ("eq", C.c_double * (NPOP * NMOM)),
    ]


def build(force: bool = False) -> None:
    """Run oracle/Makefile (needs /root/reference only for the _ref target)."""
    if force or not os.path.exists(ORC_SO) or not os.path.exists(REF_SO):
        subprocess.run(["make", "-C", HERE, "-s"], check=True)


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            subprocess.run(["make", "-C", HERE, "-s", "_build/liborc.so"], check=True)
        lib = C.CDLL(ORC_SO)
        M = C.POINTER(OrcModel)
        sig = {
            "orc_model_d2q37": (C.c_int, [M]),
            "orc_ymirror": (None, [M, C.POINTER(C.c_int)]),
            "orc_macros": (C.c_int, [M, _dp, _dp]),
            "orc_equilibrium": (None, [M, _dp, _dp]),
            "orc_collide_site": (C.c_int, [M, _dp, C.c_double, _dp]),
            "orc_propagate": (C.c_int, [M, C.c_int, C.c_int, C.c_int, _dp, _dp]),
            "orc_propagate_mt": (C.c_int, [M, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int]),
            "orc_collide": (C.c_int, [M, C.c_int, C.c_int, C.c_double, _dp, _dp, C.c_int]),
            "orc_step": (C.c_int, [M, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, _dp, _dp, C.c_int]),
            "orc_padded_elems": (C.c_size_t, [C.c_int, C.c_int, C.c_int]),
            "orc_canonical_to_padded": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp]),
            "orc_padded_to_canonical": (C.c_int, [C.c_int, C.c_int, C.c_int, _dp, _dp]),
            "orc_halo_fill": (C.c_int, [M, C.c_int, C.c_int, C.c_int, C.c_int, _dp]),
            "orc_propagate_padded": (C.c_int, [M, C.c_int, C.c_int, C.c_int, _dp, _dp]),
            "orc_mt64_fill_u01": (None, [C.c_uint64, C.c_size_t, _dp]),
            "orc_philox4x32_10": (None, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
            "orc_random_lattice": (None, [M, C.c_int, C.c_int, C.c_uint64, _dp]),
            "orc_equilibrium_lattice": (None, [M, C.c_int, C.c_int, _dp, _dp]),
            "orc_shear_lattice": (None, [M, C.c_int, C.c_int, C.c_double, C.c_double, _dp]),
            "orc_rt_lattice": (None, [M, C.c_int, C.c_int, C.c_uint64, _dp]),
            "orc_c2_lattice": (None, [M, C.c_int, C.c_int, C.c_uint64, _dp]),
            "orc_rt_philox_lattice": (None, [M, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, _dp]),
            "orc_philox_lattice": (None, [C.c_int, C.c_int, C.c_uint64, _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference library {REF_SO} not built (run make -C oracle)")
        lib = C.CDLL(REF_SO)
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_model": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int), _dp, C.POINTER(C.c_double), _dp]),
            "ref_macros": (C.c_int, [_dp, _dp]),
            "ref_equilibrium": (C.c_int, [_dp, _dp]),
            "ref_collide_site": (C.c_int, [_dp, C.c_double, _dp]),
            "ref_random_lattice": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _dp]),
            "ref_equilibrium_lattice": (C.c_int, [C.c_int, C.c_int, _dp, _dp]),
            "ref_shear_lattice": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, _dp]),
            "ref_oracle_propagate": (C.c_int, [C.c_int, C.c_int, _dp, _dp]),
            "ref_oracle_collide": (C.c_int, [C.c_int, C.c_int, C.c_double, _dp, _dp]),
            "ref_sim_create": (vp, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
            "ref_sim_destroy": (None, [vp]),
            "ref_sim_elems": (C.c_size_t, [vp]),
            "ref_sim_load": (C.c_int, [vp, _dp]),
            "ref_sim_load_into": (C.c_int, [vp, C.c_int, _dp]),
            "ref_sim_dump": (C.c_int, [vp, C.c_int, _dp]),
            "ref_sim_read_raw": (C.c_int, [vp, C.c_int, _dp]),
            "ref_sim_halo_exchange": (C.c_int, [vp]),
            "ref_sim_propagate": (C.c_int, [vp, C.c_int]),
            "ref_sim_collide": (C.c_int, [vp, C.c_double]),
            "ref_sim_step": (C.c_int, [vp, C.c_double, C.c_int, C.c_int]),
            "ref_sim_time_step_counter": (C.c_long, [vp]),
            "ref_sim_time": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
            "ref_hardware_concurrency": (C.c_int, []),
            "ref_save_dump": (C.c_int, [C.c_int, C.c_int, _dp, C.c_char_p]),
            "ref_load_dump": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.c_void_p, C.c_size_t]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _ref = lib
    return _ref


# --------------------------------------------------------------------------- model

class Model:
    """Velocity set, weights, t0 and Hermite table from one of the two oracles."""

    def __init__(self, cx, cy, w, t0, eq):
        self.cx = np.asarray(cx, dtype=np.int32)
        self.cy = np.asarray(cy, dtype=np.int32)
        self.w = np.asarray(w, dtype=np.float64)
        self.t0 = float(t0)
        self.eq = np.asarray(eq, dtype=np.float64).reshape(NPOP, NMOM)

    def ymirror(self) -> np.ndarray:
        out = np.empty(NPOP, dtype=np.int64)
        for p in range(NPOP):
            out[p] = int(np.nonzero((self.cx == self.cx[p]) & (self.cy == -self.cy[p]))[0][0])
        return out


_orc_model = None


def orc_model_struct() -> OrcModel:
    global _orc_model
    if _orc_model is None:
        m = OrcModel()
        if orc().orc_model_d2q37(C.byref(m)) != 0:
            raise RuntimeError("oracle weight derivation failed")
        _orc_model = m
    return _orc_model


def orc_model() -> Model:
    m = orc_model_struct()
    return Model(list(m.cx), list(m.cy), list(m.w), m.t0, list(m.eq))


def ref_model() -> Model:
    cx = (C.c_int * NPOP)()
    cy = (C.c_int * NPOP)()
    w = np.empty(NPOP)
    t0 = C.c_double()
    eq = np.empty(NPOP * NMOM)
    if ref().ref_model(cx, cy, w, C.byref(t0), eq) != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return Model(list(cx), list(cy), w, t0.value, eq)


# --------------------------------------------------------------------------- oracle (C restatement)

def _canon(lx, ly):
    return np.empty((NPOP, lx, ly), dtype=np.float64)


def _flat(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(-1), a


def orc_propagate(a, bc=BC_PERIODIC, nthreads=None):
    _, lx, ly = a.shape
    fa, _ = _flat(a)
    out = _canon(lx, ly)
    if orc().orc_propagate_mt(C.byref(orc_model_struct()), lx, ly, bc, fa, out.reshape(-1),
                              nthreads or os.cpu_count() or 1) != 0:
        raise ValueError("orc_propagate: bad geometry")
    return out


def orc_collide(a, omega, nthreads=None):
    _, lx, ly = a.shape
    fa, _ = _flat(a)
    out = _canon(lx, ly)
    bad = orc().orc_collide(C.byref(orc_model_struct()), lx, ly, float(omega), fa, out.reshape(-1),
                            nthreads or os.cpu_count() or 1)
    return out, bool(bad)


def orc_step(a, omega, nsteps, bc=BC_PERIODIC, nthreads=None):
    _, lx, ly = a.shape
    st = np.array(a, dtype=np.float64, copy=True)
    scratch = _canon(lx, ly)
    rc = orc().orc_step(C.byref(orc_model_struct()), lx, ly, bc, float(omega), int(nsteps),
                        st.reshape(-1), scratch.reshape(-1), nthreads or os.cpu_count() or 1)
    if rc < 0:
        raise ValueError("orc_step: bad geometry")
    return st, bool(rc)


def orc_collide_site(f, omega):
    out = np.empty(NPOP)
    bad = orc().orc_collide_site(C.byref(orc_model_struct()), np.ascontiguousarray(f, dtype=np.float64),
                                 float(omega), out)
    return out, bool(bad)


def orc_macros(f):
    mac = np.empty(4)
    bad = orc().orc_macros(C.byref(orc_model_struct()), np.ascontiguousarray(f, dtype=np.float64), mac)
    return mac, bool(bad)


def orc_equilibrium(mac):
    out = np.empty(NPOP)
    orc().orc_equilibrium(C.byref(orc_model_struct()), np.ascontiguousarray(mac, dtype=np.float64), out)
    return out


def padded_elems(lx, ly, vl):
    return int(orc().orc_padded_elems(lx, ly, vl))


def orc_to_padded(a, vl):
    _, lx, ly = a.shape
    out = np.zeros(padded_elems(lx, ly, vl))
    fa, _ = _flat(a)
    if orc().orc_canonical_to_padded(lx, ly, vl, fa, out) != 0:
        raise ValueError("bad padded geometry")
    return out


def orc_from_padded(buf, lx, ly, vl):
    out = _canon(lx, ly)
    if orc().orc_padded_to_canonical(lx, ly, vl, np.ascontiguousarray(buf), out.reshape(-1)) != 0:
        raise ValueError("bad padded geometry")
    return out


def orc_halo_fill(buf, lx, ly, vl, bc=BC_PERIODIC):
    buf = np.array(buf, dtype=np.float64, copy=True)
    if orc().orc_halo_fill(C.byref(orc_model_struct()), lx, ly, vl, bc, buf) != 0:
        raise ValueError("bad padded geometry")
    return buf


def orc_propagate_padded(buf, lx, ly, vl):
    out = np.zeros_like(buf)
    if orc().orc_propagate_padded(C.byref(orc_model_struct()), lx, ly, vl, np.ascontiguousarray(buf), out) != 0:
        raise ValueError("bad padded geometry")
    return out


def mt64_u01(seed, n):
    out = np.empty(n)
    orc().orc_mt64_fill_u01(seed, n, out)
    return out


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    orc().orc_philox4x32_10(c, k, o)
    return list(o)


def orc_lattice(kind, lx, ly, seed=12345, **kw):
    """Initialisers: random (lattice.cpp:8-23), equilibrium, shear, rt (c0), c2, philox (c1)."""
    out = _canon(lx, ly)
    M = C.byref(orc_model_struct())
    o = out.reshape(-1)
    if kind == "random":
        orc().orc_random_lattice(M, lx, ly, seed, o)
    elif kind == "equilibrium":
        orc().orc_equilibrium_lattice(M, lx, ly, np.asarray(kw["mac"], dtype=np.float64), o)
    elif kind == "shear":
        orc().orc_shear_lattice(M, lx, ly, kw.get("amp", 0.02), kw["temp"], o)
    elif kind == "rt":
        orc().orc_rt_lattice(M, lx, ly, seed, o)
    elif kind == "c2":
        orc().orc_c2_lattice(M, lx, ly, seed, o)
    elif kind == "rt_philox":
        orc().orc_rt_philox_lattice(M, lx, ly, kw.get("ly_global", ly), kw.get("y0", 0), seed, o)
    elif kind == "philox":
        orc().orc_philox_lattice(lx, ly, seed, o)
    else:
        raise ValueError(kind)
    return out


# --------------------------------------------------------------------------- reference (compiled)

def _ref_check(rc):
    if rc != 0:
        msg = ref().ref_last_error().decode()
        if rc == 2:
            raise FloatingPointError("NonPhysicalError: " + msg)
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def ref_random_lattice(lx, ly, seed):
    out = _canon(lx, ly)
    _ref_check(ref().ref_random_lattice(lx, ly, seed, out.reshape(-1)))
    return out


def ref_oracle_propagate(a):
    _, lx, ly = a.shape
    out = _canon(lx, ly)
    fa, _ = _flat(a)
    _ref_check(ref().ref_oracle_propagate(lx, ly, fa, out.reshape(-1)))
    return out


def ref_oracle_collide(a, omega):
    _, lx, ly = a.shape
    out = _canon(lx, ly)
    fa, _ = _flat(a)
    _ref_check(ref().ref_oracle_collide(lx, ly, float(omega), fa, out.reshape(-1)))
    return out


def ref_save_dump(a, path):
    """The reference's save_dump (dump.cpp:44-58)."""
    _, lx, ly = a.shape
    fa, _ = _flat(a)
    _ref_check(ref().ref_save_dump(lx, ly, fa, os.fsencode(path)))


def ref_load_dump(path):
    """The reference's load_dump (dump.cpp:60-70) -> canonical (37, lx, ly)."""
    dims = (C.c_int * 3)()
    _ref_check(ref().ref_load_dump(os.fsencode(path), dims, None, 0))
    out = np.empty((dims[2], dims[0], dims[1]))
    _ref_check(ref().ref_load_dump(os.fsencode(path), dims, out.ctypes.data, out.size))
    return out


class RefSim:
    """The reference LatticeState + ThreadPool (kernels.hpp verbs)."""

    def __init__(self, layout, lx, ly, vl=1, workers=1):
        self.lx, self.ly, self.vl = lx, ly, vl
        self.h = ref().ref_sim_create(layout, lx, ly, vl, workers)
        if not self.h:
            raise ValueError(ref().ref_last_error().decode())

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            ref().ref_sim_destroy(h)
            self.h = None

    def load(self, a, which=0):
        fa, _ = _flat(a)
        _ref_check(ref().ref_sim_load_into(self.h, which, fa))

    def dump(self, which=0):
        out = _canon(self.lx, self.ly)
        _ref_check(ref().ref_sim_dump(self.h, which, out.reshape(-1)))
        return out

    def raw(self, which=0):
        out = np.empty(ref().ref_sim_elems(self.h))
        _ref_check(ref().ref_sim_read_raw(self.h, which, out))
        return out

    def halo_exchange(self):
        _ref_check(ref().ref_sim_halo_exchange(self.h))

    def propagate(self, nt=False):
        _ref_check(ref().ref_sim_propagate(self.h, int(nt)))

    def collide(self, omega):
        _ref_check(ref().ref_sim_collide(self.h, float(omega)))

    def step(self, omega, n=1, nt=False):
        _ref_check(ref().ref_sim_step(self.h, float(omega), int(n), int(nt)))

    @property
    def time_step(self):
        return int(ref().ref_sim_time_step_counter(self.h))

    def time(self, kernel, omega=1.0, iterations=5, warmup=1, nt=False):
        med = C.c_double()
        mn = C.c_double()
        k = {"propagate": 0, "collide": 1, "step": 2}[kernel]
        _ref_check(ref().ref_sim_time(self.h, k, float(omega), iterations, warmup, int(nt),
                                      C.byref(med), C.byref(mn)))
        return med.value, mn.value
