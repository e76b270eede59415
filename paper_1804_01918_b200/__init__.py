"""B200-native D2Q37 lattice Boltzmann hot path (propagate / bc / collide / step).

Host-side Python mirror of the reference's operator API
(``/root/reference/proj/bindings/module.cpp:44-226``,
``proj/python/lbmbench/__init__.py``) over the C-ABI library
``lib/libd2q37_b200.so`` (``include/d2q37_b200.h``).  Every verb runs the
sm_100a kernels; there is no CPU fallback: if the library is missing the
import fails loudly.

Same names and argument meaning as the reference module:

* ``model()`` -> ``Model`` (npop, t0, halo_extent, velocities, weights,
  macros, equilibrium, collide_site) -- host-side per-site helpers, as in
  ``module.cpp:135-170``.
* ``Simulation(layout, lx, ly, vl=1, ...)`` with ``load``, ``dump``,
  ``init_random``, ``init_equilibrium``, ``init_shear``, ``step(omega, n)``,
  ``propagate()``, ``time_step`` (``module.cpp:44-99``); the reference's
  ``workers``/``schedule`` thread-pool arguments are accepted and ignored
  (the CUDA grid replaces the pool).  Extra verbs: ``bc``, ``collide``,
  ``sync``, ``moments``, ``read_padded``.
* ``mlups``, ``propagate_gbps``, ``collide_gflops`` (``metrics.cpp:50-63``).

Errors map to the reference's exception types: ``ValueError`` for
``std::invalid_argument`` and ``NonPhysicalError`` (a ``FloatingPointError``)
for ``lbm::NonPhysicalError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "NPOP", "Model", "Simulation", "SlabGroup", "NonPhysicalError", "model", "mlups",
    "propagate_gbps", "collide_gflops", "make_lattice", "library_path", "nccl_unique_id",
    "COLLIDE_FLOPS_PER_SITE", "__version__", "convert", "scalar_steps", "p2p_ring", "step_slabs", "MultiGPU",
]
__version__ = "0.1.0"

NPOP = 37
NMOM = 14
HALO = 3
COLLIDE_FLOPS_PER_SITE = 1522  # VelocityModel::kCollideFlopsPerSite (model.hpp:74-78)

OK, ERR_INVALID, ERR_NON_PHYSICAL, ERR_CUDA, ERR_NCCL, ERR_UNSUPPORTED = range(6)
LAYOUTS = {"aos": 0, "soa": 1, "csoa": 2, "caosoa": 3, "banded": 4}  # banded: the FUSED2 device store
BCS = {"periodic": 0, "wall": 1}
VARIANTS = {"unfused": 0, "fused": 1, "fused2": 2}
MATHS = {"fast": 0, "strict": 1}
INITS = {"random": 0, "equilibrium": 1, "shear": 2, "rt": 3, "c2": 4, "philox": 5}

_HERE = os.path.dirname(os.path.abspath(__file__))


def library_path() -> str:
    """The in-tree build, or D2Q37_LIBRARY (A/B runs of another build of the same library)."""
    return os.environ.get("D2Q37_LIBRARY") or os.path.join(_HERE, "lib", "libd2q37_b200.so")


class NonPhysicalError(FloatingPointError):
    """lbm::NonPhysicalError (model.hpp:28-30): a site had !(rho > 0)."""


class CudaError(RuntimeError):
    pass


class _Model(C.Structure):
    _fields_ = [
        ("cx", C.c_int * NPOP),
        ("cy", C.c_int * NPOP),
        ("w", C.c_double * NPOP),
        ("t0", C.c_double),
        ("eq", C.c_double * (NPOP * NMOM)),
    ]


_lib = None
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C {os.path.join(_HERE, 'csrc')}` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    vp, i, d, sz = C.c_void_p, C.c_int, C.c_double, C.c_size_t
    P = C.POINTER
    sig = {
        "d2q37_last_error": (C.c_char_p, []),
        "d2q37_model_d2q37": (i, [P(_Model)]),
        "d2q37_create": (i, [i, i, i, i, i, P(vp)]),
        "d2q37_destroy": (i, [vp]),
        "d2q37_set_model": (i, [vp, P(_Model)]),
        "d2q37_set_math": (i, [vp, i]),
        "d2q37_set_stream": (i, [vp, vp]),
        "d2q37_get_stream": (vp, [vp]),
        "d2q37_geometry": (i, [vp, P(C.c_int)]),
        "d2q37_device_bytes": (sz, [vp]),
        "d2q37_time_step": (C.c_long, [vp]),
        "d2q37_load_canonical": (i, [vp, vp, sz]),
        "d2q37_dump_canonical": (i, [vp, vp, sz]),
        "d2q37_run_canonical": (i, [vp, vp, vp, sz, d, i, i, i]),
        "d2q37_last_run_mode": (i, [vp]),
        "d2q37_debug_stream_plan": (i, [i, i, i, P(C.c_int), i]),
        "d2q37_load_buffer": (i, [vp, i, vp, sz]),
        "d2q37_dump_buffer": (i, [vp, i, vp, sz]),
        "d2q37_load_buffer_device": (i, [vp, i, vp, sz]),
        "d2q37_dump_buffer_device": (i, [vp, i, vp, sz]),
        "d2q37_read_padded": (i, [vp, i, _dp, sz]),
        "d2q37_write_padded": (i, [vp, i, _dp, sz]),
        "d2q37_bc": (i, [vp, i]),
        "d2q37_propagate": (i, [vp]),
        "d2q37_propagate_corrupt": (i, [vp, i]),
        "d2q37_collide": (i, [vp, d]),
        "d2q37_step": (i, [vp, d, i, i, i]),
        "d2q37_sync": (i, [vp]),
        "d2q37_swap_buffers": (i, [vp]),
        "d2q37_moments": (i, [vp, _dp]),
        "d2q37_make_lattice": (i, [i, i, i, C.c_uint64, vp, P(_Model), vp, sz, i]),
        "d2q37_fill_philox": (i, [vp, i, C.c_uint64]),
        "d2q37_init_rt_device": (i, [vp, C.c_uint64]),
        "d2q37_save_dump": (i, [vp, C.c_char_p]),
        "d2q37_load_dump": (i, [vp, C.c_char_p]),
        "d2q37_nccl_unique_id": (i, [C.c_char_p]),
        "d2q37_create_slab": (i, [i, i, i, i, i, i, i, C.c_char_p, P(vp)]),
        "d2q37_create_group": (i, [i, i, i, i, i, i, P(vp)]),
        "d2q37_group_step": (i, [P(vp), i, d, i, i, i]),
        "d2q37_slab_info": (i, [vp, P(C.c_int)]),
        "d2q37_halo_plan": (i, [P(C.c_int)] * 4),
        "d2q37_slab_neighbors": (i, [i, i, i, P(C.c_int)]),
        "d2q37_exposed_halo_ms": (d, [vp]),
        "d2q37_set_profiling": (i, [vp, i]),
        "d2q37_kernel_times": (i, [vp, _dp, P(C.c_long)]),
        "d2q37_convert": (i, [vp, vp]),
        "d2q37_create_slab_p2p": (i, [i, i, i, i, i, i, i, P(vp)]),
        "d2q37_create_multi": (i, [i, i, i, i, i, P(C.c_int), P(vp)]),
        "d2q37_multi_step": (i, [P(vp), i, d, i, i, i]),
        "d2q37_p2p_export": (i, [vp, C.c_char_p]),
        "d2q37_p2p_connect": (i, [vp, C.c_char_p, C.c_char_p]),
        "d2q37_scalar_steps": (i, [P(_Model), i, i, vp, vp, sz, d, i, i, i]),
        "d2q37_fp64_peak": (i, [i, P(C.c_double)]),
        "d2q37_set_fused2_tuning": (i, [i, i, P(C.c_int), P(C.c_int)]),
        "d2q37_set_fused2_schedule": (i, [i, P(C.c_int)]),
        "d2q37_debug_step2_slab_sweep": (i, [vp, d, i, i, i]),
        "d2q37_slab_timeline": (i, [vp, P(d)]),
        "d2q37_debug_read_halo6": (i, [vp, i, P(d), sz]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def stream_plan(ly: int, nsteps: int, bc: str = "wall") -> np.ndarray:
    """Test hook (d2q37_debug_stream_plan, no GPU needed): the operations of a pipelined run() as an
    (n, 4) int array of {kind, a, b, c}; empty when the call would run the three verbs."""
    lib = _load()
    n = lib.d2q37_debug_stream_plan(int(ly), int(nsteps), BCS[bc], None, 0)
    if n < 0:
        _check(-n)
    out = np.zeros((max(n, 0), 4), dtype=np.int32)
    if n > 0:
        lib.d2q37_debug_stream_plan(int(ly), int(nsteps), BCS[bc], out.ctypes.data_as(C.POINTER(C.c_int)), n)
    return out


def _check(rc: int) -> None:
    if rc == OK:
        return
    msg = _load().d2q37_last_error().decode()
    if rc == ERR_NON_PHYSICAL:
        raise NonPhysicalError(msg)
    if rc in (ERR_INVALID, ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(f"d2q37 error {rc}: {msg}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------------- model

class Model:
    """VelocityModel::d2q37() (model.hpp:52-72), derived by the library's host code.

    ``macros`` / ``equilibrium`` / ``collide_site`` are host-side per-site
    helpers (numpy, reference operation order) for inspection and tests; the
    lattice-wide arithmetic runs on the GPU.
    """

    npop = NPOP
    halo_extent = HALO
    collide_flops_per_site = COLLIDE_FLOPS_PER_SITE

    def __init__(self, struct: _Model | None = None):
        if struct is None:
            struct = _Model()
            _check(_load().d2q37_model_d2q37(C.byref(struct)))
        self._s = struct
        self.velocities = np.stack([np.array(struct.cx[:]), np.array(struct.cy[:])], axis=1).astype(np.int32)
        self.weights = np.array(struct.w[:], dtype=np.float64)
        self.t0 = float(struct.t0)
        self.eq_table = np.array(struct.eq[:], dtype=np.float64).reshape(NPOP, NMOM)

    @classmethod
    def from_arrays(cls, cx, cy, w, t0, eq) -> "Model":
        s = _Model()
        s.cx[:] = [int(v) for v in cx]
        s.cy[:] = [int(v) for v in cy]
        s.w[:] = [float(v) for v in w]
        s.t0 = float(t0)
        s.eq[:] = [float(v) for v in np.asarray(eq, dtype=np.float64).reshape(-1)]
        return cls(s)

    def macros(self, f):
        f = np.asarray(f, dtype=np.float64)
        c = self.velocities.astype(np.float64)
        rho = 0.0
        for v in f:
            rho += v
        if not rho > 0.0:
            raise NonPhysicalError("non-positive density")
        jx = jy = e2 = 0.0
        for i in range(NPOP):
            jx += c[i, 0] * f[i]
        for i in range(NPOP):
            jy += c[i, 1] * f[i]
        for i in range(NPOP):
            e2 += (c[i, 0] ** 2 + c[i, 1] ** 2) * f[i]
        inv = 1.0 / rho
        ux, uy = jx * inv, jy * inv
        return rho, ux, uy, 0.5 * (e2 * inv - (ux * ux + uy * uy))

    def equilibrium(self, rho, ux, uy, temp):
        dt = temp - self.t0
        ux2, uy2, uxuy = ux * ux, uy * uy, ux * uy
        dt3, dt6, dt2 = 3.0 * dt, 6.0 * dt, dt * dt
        dt2x3 = 3.0 * dt2
        mom = np.array([ux, uy, ux2 + dt, uxuy, uy2 + dt, ux * (ux2 + dt3), uy * (ux2 + dt),
                        ux * (uy2 + dt), uy * (uy2 + dt3), ux2 * (ux2 + dt6) + dt2x3,
                        uxuy * (ux2 + dt3), uxuy * uxuy + dt * (ux2 + uy2) + dt2,
                        uxuy * (uy2 + dt3), uy2 * (uy2 + dt6) + dt2x3])
        out = np.empty(NPOP)
        for i in range(NPOP):
            s = 1.0
            for k in range(NMOM):
                s += self.eq_table[i, k] * mom[k]
            out[i] = rho * self.weights[i] * s
        return out

    def collide_site(self, f, omega):
        f = np.asarray(f, dtype=np.float64)
        feq = self.equilibrium(*self.macros(f))
        return f + omega * (feq - f)

    def ymirror(self) -> np.ndarray:
        v = self.velocities
        return np.array([int(np.nonzero((v[:, 0] == v[p, 0]) & (v[:, 1] == -v[p, 1]))[0][0])
                         for p in range(NPOP)])


_default_model = None


def model() -> Model:
    """The D2Q37 model singleton (module.cpp:172)."""
    global _default_model
    if _default_model is None:
        _default_model = Model()
    return _default_model


# --------------------------------------------------------------------------- metrics (metrics.cpp:50-63)

def mlups(lx: int, ly: int, t_iter_s: float) -> float:
    if not t_iter_s > 0.0:
        raise ValueError("iteration time must be positive")
    return float(lx) * ly / (t_iter_s * 1e6)


def propagate_gbps(lx: int, ly: int, npop: int, t_iter_s: float, traffic: str = "nt") -> float:
    if not t_iter_s > 0.0:
        raise ValueError("iteration time must be positive")
    k = {"nt": 2, "rfo": 3}[traffic]
    return float(lx) * ly * npop * 8.0 * k / (t_iter_s * 1e9)


def collide_gflops(lx: int, ly: int, flops_per_site: float, t_iter_s: float) -> float:
    if not t_iter_s > 0.0:
        raise ValueError("iteration time must be positive")
    return float(lx) * ly * flops_per_site / (t_iter_s * 1e9)


# --------------------------------------------------------------------------- initialisers

def make_lattice(kind: str, lx: int, ly: int, seed: int = 12345, params=None, mdl: Model | None = None,
                 nthreads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    """Host generators (lattice.cpp:8-47 + BASELINE recipes) -> canonical (37, lx, ly)."""
    if out is None:
        out = np.empty((NPOP, lx, ly), dtype=np.float64)
    if out.shape != (NPOP, lx, ly) or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous float64 array of shape (37, lx, ly)")
    par = None
    if params is not None:
        par = np.ascontiguousarray(params, dtype=np.float64)
    m = (mdl or model())._s
    _check(_load().d2q37_make_lattice(INITS[kind], lx, ly, seed, None if par is None else _ptr(par),
                                      C.byref(m), _ptr(out), out.size, nthreads))
    return out


def scalar_steps(canon, omega: float, nsteps: int, math: str = "fast", mdl: Model | None = None,
                 device: int = 0) -> np.ndarray:
    """The scalar device reference of run_validation (validation.cpp:13-38): ``nsteps`` of
    propagate then collide, periodic in x and y, on a halo-free canonical array with explicit
    modulo indexing (d2q37_scalar_steps).  Returns a new (37, lx, ly) array."""
    a = np.ascontiguousarray(canon, dtype=np.float64)
    if a.ndim != 3 or a.shape[0] != NPOP:
        raise ValueError("canonical array must have shape (37, lx, ly)")
    out = np.empty_like(a)
    m = (mdl or model())._s
    _check(_load().d2q37_scalar_steps(C.byref(m), a.shape[1], a.shape[2], _ptr(a), _ptr(out), a.size,
                                      float(omega), int(nsteps), MATHS[math], device))
    return out


def convert(src: "Simulation", layout: str, vl: int = 1) -> "Simulation":
    """convert(src, to) (layout.hpp:148, layout.cpp:105-116): a new lattice with ``layout``/``vl``
    holding the physical sites of ``src``'s state buffer, on the same device."""
    dst = Simulation(layout, src.lx, src.ly, vl, device=src.device, bc=src.bc_mode, variant=src.variant,
                     math=src.math, mdl=src.model)
    _check(_load().d2q37_convert(src._h, dst._h))
    return dst


def halo_plan():
    """(lo_entries, hi_entries): lists of (d, p) of the slab halo messages (d2q37_halo_plan)."""
    arrs = [(C.c_int * 32)() for _ in range(4)]
    n = _load().d2q37_halo_plan(*arrs)
    if n < 0:
        raise RuntimeError("asymmetric halo plan")
    lo = [(arrs[0][i], arrs[1][i]) for i in range(n)]
    hi = [(arrs[2][i], arrs[3][i]) for i in range(n)]
    return lo, hi


def slab_neighbors(rank: int, nranks: int, bc: str = "periodic"):
    """(lo_peer, hi_peer) of a y-slab rank; -1 where the face is a wall."""
    out = (C.c_int * 2)()
    _check(_load().d2q37_slab_neighbors(rank, nranks, BCS[bc], out))
    return out[0], out[1]


def fp64_peak(device: int = 0) -> float:
    """Achieved FP64 TFLOP/s of independent DFMA chains on every SM (the FP64 roofline denominator
    at the clocks the GPU holds under load; MEASURED_PEAKS.json has no FP64 figure)."""
    out = C.c_double(0.0)
    _check(_load().d2q37_fp64_peak(int(device), C.byref(out)))
    return out.value


def set_fused2_tuning(form: int = -1, face_pct: int = -1) -> tuple:
    """Process-wide FUSED2 tuning (d2q37_set_fused2_tuning): ``form`` 0 = per-thread loads, 1 / 2 =
    interior bands staged by one bulk-copy stage, 3 = two stages, 4 = two stages and two threads per
    site (default; all bit-identical); ``face_pct`` sizes the face-band CTA
    groups (0 = the form's default).  -1 leaves a setting unchanged.  Returns the previous
    (form, face_pct)."""
    pf, pp = C.c_int(0), C.c_int(0)
    _check(_load().d2q37_set_fused2_tuning(int(form), int(face_pct), C.byref(pf), C.byref(pp)))
    return pf.value, pp.value


def set_fused2_schedule(sched: int = -1) -> int:
    """Process-wide FUSED2 interior schedule (d2q37_set_fused2_schedule): 1 = lockstep (default; CTAs
    of neighbouring bands march the same columns together), 0 = band-major item ranges.  Both are
    bit-identical.  -1 leaves it unchanged.  Returns the previous schedule."""
    prev = C.c_int(0)
    _check(_load().d2q37_set_fused2_schedule(int(sched), C.byref(prev)))
    return prev.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_load().d2q37_nccl_unique_id(buf))
    return buf.raw


def p2p_ring(layout: str, lx: int, ly: int, vl: int = 1, nslabs: int = 2, *, device: int = 0,
             bc: str = "periodic", variant: str = "fused", math: str = "fast") -> list:
    """``nslabs`` P2P y-slabs of one lattice in this process, connected as a ring (the same
    peer-memory halo protocol as one slab per GPU; here every neighbour is in this process).
    Step them together with :func:`step_slabs`."""
    slabs = [Simulation.slab(layout, lx, ly, vl, device=device, rank=r, nranks=nslabs, bc=bc, variant=variant,
                             math=math, transport="p2p")
             for r in range(nslabs)]
    if nslabs > 1:
        blobs = [s.p2p_blob() for s in slabs]
        for r, s in enumerate(slabs):
            s.p2p_connect(blobs[(r - 1) % nslabs], blobs[(r + 1) % nslabs])
    return slabs


def step_slabs(slabs, omega: float, n: int = 1):
    """Advance in-process slabs in lockstep (one step each, rank order), then sync them."""
    for _ in range(n):
        for s in slabs:
            s.step(omega, 1, sync=False)
    for s in slabs:
        s.sync()


# --------------------------------------------------------------------------- lattice

class Simulation:
    """One device lattice (LatticeState + kernels.hpp verbs) -- module.cpp:44-99.

    ``bc``: "periodic" (reference halo_exchange) or "wall" (top/bottom
    specular walls, BASELINE config 0).  ``variant``: "fused" or "unfused"
    step.  ``math``: "fast" (DFMA contraction) or "strict" (IEEE op per op).
    """

    def __init__(self, layout: str, lx: int, ly: int, vl: int = 1, workers: int = 1,
                 schedule: str = "dynamic", *, device: int = 0, bc: str = "periodic",
                 variant: str = "fused", math: str = "fast", mdl: Model | None = None,
                 _handle=None):
        lib = _load()
        if layout not in LAYOUTS:
            raise ValueError(f"unknown layout: {layout}")
        if schedule not in ("dynamic", "static"):
            raise ValueError(f"unknown schedule: {schedule}")
        if workers < 1:
            raise ValueError("worker count must be >= 1")
        self.layout, self.bc_mode, self.variant = layout, bc, variant
        self.device, self.math = device, math
        if _handle is None:
            h = C.c_void_p()
            _check(lib.d2q37_create(LAYOUTS[layout], lx, ly, vl, device, C.byref(h)))
            self._h = h
        else:
            self._h = _handle
        g = (C.c_int * 6)()
        _check(lib.d2q37_geometry(self._h, g))
        self.lx, self.ly, self.vl, self.strip, self.sy, self.px = list(g)
        self.model = mdl or model()
        _check(lib.d2q37_set_model(self._h, C.byref(self.model._s)))
        self.set_math(math)
        self._owned = _handle is None

    @classmethod
    def slab(cls, layout: str, lx: int, ly_global: int, vl: int = 1, *, device: int = 0, rank: int = 0,
             nranks: int = 1, nccl_id: bytes | None = None, bc: str = "periodic", variant: str = "fused",
             math: str = "fast", mdl: Model | None = None, transport: str = "nccl",
             exchange=None) -> "Simulation":
        """Rank `rank` of an `nranks`-GPU y-slab decomposition.

        ``transport="nccl"`` (d2q37_create_slab): NCCL send/recv halos; needs ``nccl_id``.
        ``transport="p2p"`` (d2q37_create_slab_p2p): the step kernel pushes its face sites into
        the neighbours' ghost slots through peer memory.
        ``exchange(blob) -> list of every rank's blob`` (e.g. an all_gather over
        torch.distributed) connects the ranks; with ``nranks == 1`` and no ``exchange`` the slab
        is a 1-rank ring connected to itself.  Without either, call ``p2p_blob`` /
        ``p2p_connect`` yourself."""
        h = C.c_void_p()
        if transport == "p2p":
            _check(_load().d2q37_create_slab_p2p(LAYOUTS[layout], lx, ly_global, vl, device, rank, nranks,
                                                 C.byref(h)))
        elif transport == "nccl":
            _check(_load().d2q37_create_slab(LAYOUTS[layout], lx, ly_global, vl, device, rank, nranks,
                                             nccl_id, C.byref(h)))
        else:
            raise ValueError(f"unknown transport: {transport}")
        sim = cls(layout, lx, ly_global // nranks, vl, device=device, bc=bc, variant=variant, math=math,
                  mdl=mdl, _handle=h)
        sim._owned = True
        sim.rank, sim.nranks, sim.transport = rank, nranks, transport
        if transport == "p2p":
            if exchange is not None:
                blobs = list(exchange(sim.p2p_blob()))
                sim.p2p_connect(blobs[(rank - 1) % nranks], blobs[(rank + 1) % nranks])
            elif nranks == 1:
                b = sim.p2p_blob()
                sim.p2p_connect(b, b)
        return sim

    def p2p_blob(self) -> bytes:
        """This slab's 256-byte connection blob (d2q37_p2p_export)."""
        buf = C.create_string_buffer(256)
        _check(_load().d2q37_p2p_export(self._h, buf))
        return buf.raw

    def p2p_connect(self, lo_blob: bytes | None, hi_blob: bytes | None):
        """Maps the lo / hi neighbours' buffers and step counters (d2q37_p2p_connect)."""
        _check(_load().d2q37_p2p_connect(self._h, lo_blob, hi_blob))

    def slab_info(self):
        out = (C.c_int * 4)()
        _check(_load().d2q37_slab_info(self._h, out))
        return tuple(out)

    def close(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owned", False):
            _load().d2q37_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # configuration
    def set_math(self, math: str):
        _check(_load().d2q37_set_math(self._h, MATHS[math]))
        self.math = math

    def set_model(self, mdl: Model):
        self.model = mdl
        _check(_load().d2q37_set_model(self._h, C.byref(mdl._s)))

    @property
    def stream(self) -> int:
        return _load().d2q37_get_stream(self._h) or 0

    def set_stream(self, stream_ptr: int):
        _check(_load().d2q37_set_stream(self._h, C.c_void_p(stream_ptr)))

    @property
    def device_bytes(self) -> int:
        return int(_load().d2q37_device_bytes(self._h))

    @property
    def time_step(self) -> int:
        return int(_load().d2q37_time_step(self._h))

    @property
    def shape(self):
        return (NPOP, self.lx, self.ly)

    # state (lattice.hpp:18-19, dump.hpp:28-29)
    def _canon_in(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        if a.ndim != 3 or a.shape[0] != NPOP:
            raise ValueError("expected an array of shape (37, lx, ly)")
        return a

    def load(self, arr, which: int = 0):
        a = self._canon_in(arr)
        _check(_load().d2q37_load_buffer(self._h, which, _ptr(a), a.size))

    def dump(self, which: int = 0, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.shape, dtype=np.float64)
        if out.shape != self.shape or not out.flags.c_contiguous or out.dtype != np.float64:
            raise ValueError("out must be a C-contiguous float64 (37, lx, ly) array")
        _check(_load().d2q37_dump_buffer(self._h, which, _ptr(out), out.size))
        return out

    def run(self, arr, omega: float = 1.0, n: int = 1, *, out: np.ndarray | None = None, bc: str | None = None,
            variant: str | None = None) -> np.ndarray:
        """load(arr) + step(omega, n) + dump(out) in one call (d2q37_run_canonical), bit-identical to the
        three verbs; on a single SoA wall domain with FUSED2 and an even n the copies are pipelined in
        y-chunks under the sweeps.  ``out`` may be ``arr`` itself (pinned host memory overlaps best)."""
        a = self._canon_in(arr)
        if a.shape != self.shape:
            raise ValueError("expected an array of shape (37, lx, ly)")
        if out is None:
            out = np.empty(self.shape, dtype=np.float64)
        if out.shape != self.shape or not out.flags.c_contiguous or out.dtype != np.float64:
            raise ValueError("out must be a C-contiguous float64 (37, lx, ly) array")
        _check(_load().d2q37_run_canonical(self._h, _ptr(a), _ptr(out), a.size, float(omega), int(n),
                                           VARIANTS[variant or self.variant], BCS[bc or self.bc_mode]))
        return out

    @property
    def last_run_mode(self) -> str:
        """How the last run() ran: "three_verbs", "pipelined_walls" or "pipelined_periodic"."""
        return ("three_verbs", "pipelined_walls", "pipelined_periodic")[_load().d2q37_last_run_mode(self._h)]

    def load_device(self, ptr: int, n: int, which: int = 0):
        _check(_load().d2q37_load_buffer_device(self._h, which, C.c_void_p(ptr), n))

    def dump_device(self, ptr: int, n: int, which: int = 0):
        _check(_load().d2q37_dump_buffer_device(self._h, which, C.c_void_p(ptr), n))

    def read_padded(self, which: int = 0) -> np.ndarray:
        out = np.empty(NPOP * self.px * self.sy * self.vl)
        _check(_load().d2q37_read_padded(self._h, which, out, out.size))
        return out

    def write_padded(self, buf, which: int = 0):
        b = np.ascontiguousarray(buf, dtype=np.float64)
        _check(_load().d2q37_write_padded(self._h, which, b, b.size))

    def init_random(self, seed: int):
        self.load(make_lattice("random", self.lx, self.ly, seed, mdl=self.model))

    def init_equilibrium(self, rho: float = 1.0, ux: float = 0.0, uy: float = 0.0, temp: float | None = None):
        temp = self.model.t0 if temp is None else temp
        self.load(make_lattice("equilibrium", self.lx, self.ly, params=[rho, ux, uy, temp], mdl=self.model))

    def init_shear(self, amp: float, temp: float):
        self.load(make_lattice("shear", self.lx, self.ly, params=[amp, temp], mdl=self.model))

    def init_philox(self, seed: int, which: int = 0):
        _check(_load().d2q37_fill_philox(self._h, which, seed))

    def save_dump(self, path: str):
        """save_dump (dump.cpp:44-58): LBDUMP01 file of the state, streamed from the device."""
        _check(_load().d2q37_save_dump(self._h, os.fsencode(path)))

    def load_dump(self, path: str):
        """load_dump + LatticeState::load (dump.cpp:60-70), streamed to the device."""
        _check(_load().d2q37_load_dump(self._h, os.fsencode(path)))

    def init_rt_device(self, seed: int):
        """Config-0/3/4 RT init generated on the device (Philox noise by global site)."""
        _check(_load().d2q37_init_rt_device(self._h, seed))

    # kernels (kernels.hpp:29-46); each verb is synchronous like the reference's
    def bc(self, mode: str | None = None, sync: bool = True):
        _check(_load().d2q37_bc(self._h, BCS[mode or self.bc_mode]))
        if sync:
            self.sync()

    def halo_exchange(self, sync: bool = True):
        self.bc("periodic", sync)

    def propagate_only(self, corrupt_population: int = -1, sync: bool = True):
        """propagate(prv -> nxt) without the halo fill (kernels.hpp:33)."""
        _check(_load().d2q37_propagate_corrupt(self._h, corrupt_population))
        if sync:
            self.sync()

    def propagate(self):
        """module.cpp:79-83: halo exchange + propagate, result becomes the state."""
        self.bc("periodic", sync=False)
        self.propagate_only(sync=False)
        self.swap_buffers()
        self.sync()

    def swap_buffers(self):
        """std::swap(prv, nxt) (module.cpp:82)."""
        _check(_load().d2q37_swap_buffers(self._h))

    def collide(self, omega: float, sync: bool = True):
        _check(_load().d2q37_collide(self._h, float(omega)))
        if sync:
            self.sync()

    def step(self, omega: float = 1.0, n: int = 1, *, bc: str | None = None, variant: str | None = None,
             sync: bool = True):
        _check(_load().d2q37_step(self._h, float(omega), int(n), VARIANTS[variant or self.variant],
                                  BCS[bc or self.bc_mode]))
        if sync:
            self.sync()

    def sync(self):
        _check(_load().d2q37_sync(self._h))

    KERNEL_CLASSES = ("edge", "propagate", "collide", "fused", "pack", "boundary")

    def set_profiling(self, on: bool = True):
        _check(_load().d2q37_set_profiling(self._h, int(bool(on))))

    def kernel_times(self) -> dict:
        """{class: (total_ms, launches)} since the last call (CUDA events on the lattice stream)."""
        ms = np.zeros(6)
        cnt = (C.c_long * 6)()
        _check(_load().d2q37_kernel_times(self._h, ms, cnt))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.KERNEL_CLASSES)}

    def slab_timeline(self) -> dict:
        """Last overlapped FUSED2 slab sweep with profiling on (d2q37_slab_timeline): ms after the sweep
        launch at which the exchange started / NCCL finished / the unpack finished / the sweep finished."""
        out = np.zeros(4)
        _check(_load().d2q37_slab_timeline(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return dict(zip(("exchange_start", "nccl_done", "unpack_done", "sweep_done"), out.tolist()))

    def exposed_halo_ms(self) -> float:
        return float(_load().d2q37_exposed_halo_ms(self._h))

    def debug_step2_slab_sweep(self, omega: float, form: int, face_lo: str, face_hi: str):
        """Test hook (d2q37_debug_step2_slab_sweep): one overlapped FUSED2 slab sweep with the given faces
        ("wall" / "ghost"; ghost rows read as they stand, nothing exchanged), form 4 = pair form."""
        f = {"wall": 1, "ghost": 3}
        _check(_load().d2q37_debug_step2_slab_sweep(self._h, float(omega), int(form), f[face_lo], f[face_hi]))

    def debug_read_halo6(self, which: int) -> np.ndarray:
        """Test hook: FUSED2 halo send buffer `which` (0 low, 1 high) as [37][lx][6]."""
        out = np.empty((37, self.lx, 6))
        _check(_load().d2q37_debug_read_halo6(self._h, int(which), out.ctypes.data_as(C.POINTER(C.c_double)),
                                              out.size))
        return out

    def moments(self) -> np.ndarray:
        out = np.empty(4)
        _check(_load().d2q37_moments(self._h, out))
        return out


class SlabGroup:
    """``nslabs`` y-slabs of one lattice on one device (d2q37_create_group).

    Exercises the multi-GPU schedule -- pack, exchange, local/remote edge,
    interior/boundary split -- with device copies standing in for NCCL.
    """

    def __init__(self, layout: str, lx: int, ly: int, vl: int = 1, nslabs: int = 2, *, device: int = 0,
                 bc: str = "periodic", variant: str = "fused", math: str = "fast", mdl: Model | None = None):
        lib = _load()
        hs = (C.c_void_p * nslabs)()
        _check(lib.d2q37_create_group(LAYOUTS[layout], lx, ly, vl, device, nslabs, hs))
        self._hs = hs
        self.slabs = [Simulation(layout, lx, ly // nslabs, vl, device=device, bc=bc, variant=variant,
                                 math=math, mdl=mdl, _handle=C.c_void_p(hs[r])) for r in range(nslabs)]
        self.lx, self.ly, self.nslabs = lx, ly, nslabs
        self.bc_mode, self.variant = bc, variant

    def close(self):
        for s in getattr(self, "slabs", []):
            s._h = None
        hs = getattr(self, "_hs", None)
        if hs is not None:
            for h in hs:
                if h:
                    _load().d2q37_destroy(C.c_void_p(h))
            self._hs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, arr):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        ny = self.ly // self.nslabs
        for r, s in enumerate(self.slabs):
            s.load(np.ascontiguousarray(a[:, :, r * ny:(r + 1) * ny]))

    def dump(self) -> np.ndarray:
        return np.concatenate([s.dump() for s in self.slabs], axis=2)

    def init_philox(self, seed: int):
        for s in self.slabs:
            s.init_philox(seed)

    def step(self, omega: float = 1.0, n: int = 1, *, bc: str | None = None, variant: str | None = None):
        # blocking: d2q37_group_step syncs every slab and reports any slab's NonPhysicalError
        _check(_load().d2q37_group_step(self._hs, self.nslabs, float(omega), int(n),
                                        VARIANTS[variant or self.variant], BCS[bc or self.bc_mode]))


class MultiGPU(SlabGroup):
    """One lattice as P2P y-slabs on several GPUs driven by this one process
    (d2q37_create_multi; SURVEY.md 8(b) ``create_multi``).  ``devices[r]`` holds slab r;
    devices may repeat (several slabs per GPU).  Same load / dump / step as SlabGroup."""

    def __init__(self, layout: str, lx: int, ly: int, vl: int = 1, devices=(0, 0), *, bc: str = "periodic",
                 variant: str = "fused", math: str = "fast", mdl: Model | None = None):
        lib = _load()
        n = len(devices)
        hs = (C.c_void_p * n)()
        devs = (C.c_int * n)(*[int(v) for v in devices])
        _check(lib.d2q37_create_multi(LAYOUTS[layout], lx, ly, vl, n, devs, hs))
        self._hs = hs
        self.slabs = [Simulation(layout, lx, ly // n, vl, device=int(devices[r]), bc=bc, variant=variant,
                                 math=math, mdl=mdl, _handle=C.c_void_p(hs[r])) for r in range(n)]
        self.lx, self.ly, self.nslabs, self.devices = lx, ly, n, list(devices)
        self.bc_mode, self.variant = bc, variant

    def step(self, omega: float = 1.0, n: int = 1, *, bc: str | None = None, variant: str | None = None):
        _check(_load().d2q37_multi_step(self._hs, self.nslabs, float(omega), int(n),
                                        VARIANTS[variant or self.variant], BCS[bc or self.bc_mode]))
