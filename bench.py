#!/usr/bin/env python3
"""D2Q37 FP64 hot-path benchmark (BASELINE.json metric) -- one JSON line on rank 0.

Workload (BASELINE configs 3/4): a 4096 x 16384 lattice per GPU (weak
scaling; the global lattice is 4096 x 16384*N, split into y-slabs), config-0
Rayleigh-Taylor-like init, periodic x, top/bottom specular walls, omega 0.8
(SURVEY.md 0.5).  The steps run as FUSED2 on the SoA store: every pair of
steps is one kernel that reads the lattice once and writes it two steps later
(temporal blocking, csrc/d2q37_step2.cu; bit-identical to two fused steps).
On N > 1 GPUs each rank owns a y-slab; before every two-step sweep the 6-row x
37-population halos of both faces go to the neighbours through NCCL
send/recv (pack, exchange, unpack into the deep ghost rows).
``--variant fused --layout caosoa`` selects the single-step kernel with the
peer-memory halo push instead.
value = whole-job MLUPS over the K timed steps (max over ranks of the device
time).  Inputs are larger than L2 (2 x 19.9 GB per GPU vs 126 MB), so no
explicit flush is needed.

Also reported (N=1): propagate GB/s on config 1 and collide GFLOP/s on
config 2 (the other two BASELINE metrics), the SoA/CSoA x fused/unfused
step variants, the roofline of the dominant kernel, the e2e rate through the
public API with host buffers, and the reference CPU path on this host.

``--impl reference`` times the reference's own CPU step (oracle/_ref, the
unmodified lbmbench library) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LX, LY_PER_GPU = 4096, 16384
STRONG_LY = 32768  # BASELINE config 4, strong scaling: 4096 x 32768 in total
OMEGA = 0.8
SEED = 12345
BYTES_PER_SITE = 592  # 37 x 8 B read + 37 x 8 B write (BASELINE north_star)
FLOPS_PER_SITE = 1522  # VelocityModel::kCollideFlopsPerSite (model.hpp:74-78)
HBM_NOMINAL_GBS = 8000.0  # B200 HBM3e datasheet figure (ncu's DRAM peak is ~8.2 TB/s)
FP64_NOMINAL_TFLOPS = 37.0  # B200 FP64 (CUDA cores), nominal -- no measured FP64 peak in MEASURED_PEAKS.json
METRIC = "D2Q37 FP64 MLUPS (full step: propagate + bc + collide)"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- distributed plumbing

class Dist:
    """torch.distributed plumbing (NCCL; gloo on CPU for the host-logic tests)."""

    def __init__(self, backend: str | None = None):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend or os.environ.get("BENCH_DIST_BACKEND", "gloo" if STUB else "nccl")
        self.pg = False
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if self.backend == "nccl":
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
            self.pg = True

    def _dev(self) -> str:
        return f"cuda:{self.local}" if self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.pg:
            import torch.distributed as dist
            dist.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def min(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def all_gather_bytes(self, b: bytes) -> list:
        if not self.pg:
            return [b]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, b)
        return out

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if not self.pg:
            return b
        import torch.distributed as dist
        obj = [b]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.pg:
            import torch.distributed as dist
            dist.destroy_process_group()


# --------------------------------------------------------------------------- stub backend (host-logic tests)

STUB = False  # --stub: a no-op lattice timed on the host, gloo collectives (tests/test_bench_launch.py)


class _StubSim:
    """Stands in for paper_1804_01918_b200.Simulation in --stub runs: every verb is a no-op, a step
    sleeps 50 microseconds so the timing path has something to measure."""

    host_timed = True
    stream = 0

    def __init__(self, layout, lx, ly, vl=1, *, variant="fused2", **_):
        self.layout, self.lx, self.ly, self.vl, self.variant = layout, lx, ly, vl, variant
        self._launches = 0

    def init_rt_device(self, seed):
        pass

    def step(self, omega, n=1, sync=True, **_):
        time.sleep(5e-5 * n)
        self._launches += max(1, n // 2)

    def sync(self):
        pass

    def set_profiling(self, on=True):
        pass

    def kernel_times(self):
        n, self._launches = self._launches, 0
        return {"edge": (0.0, 0), "propagate": (0.0, 0), "collide": (0.0, 0), "fused": (0.1 * n, n),
                "pack": (0.0, 0), "boundary": (0.0, 0)}

    def exposed_halo_ms(self):
        return 0.0

    def close(self):
        pass


class _StubLbm:
    class Simulation(_StubSim):
        @classmethod
        def slab(cls, layout, lx, ly_global, vl=1, *, rank=0, nranks=1, **kw):
            return cls(layout, lx, ly_global // nranks, vl, **kw)

    @staticmethod
    def nccl_unique_id():
        return b"stub"

    @staticmethod
    def fp64_peak(dev):
        raise RuntimeError("stub")


def cuda_sync():
    if not STUB:
        import torch
        torch.cuda.synchronize()


# --------------------------------------------------------------------------- GPU helpers

def cuda_events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def steps_per_call(variant: str) -> int:
    """FUSED2 advances two steps per kernel: the timed loop calls step(omega, 2)."""
    return 2 if variant == "fused2" else 1


def time_stepping(sim, steps: int, variant: str) -> float:
    """Device time (ms) of exactly `steps` time steps, issued as step(omega, 2) calls for FUSED2."""
    spc = steps_per_call(variant)
    calls = [spc] * (steps // spc) + ([steps % spc] if steps % spc else [])
    it = iter(calls)
    return time_steps(sim, len(calls), lambda: sim.step(OMEGA, next(it), sync=False))


def time_steps(sim, steps: int, fn) -> float:
    """Device time (ms) of `steps` calls of fn on the lattice stream (CUDA events)."""
    if getattr(sim, "host_timed", False):  # --stub
        t0 = time.perf_counter()
        for _ in range(steps):
            fn()
        return 1e3 * (time.perf_counter() - t0)
    import torch
    s = torch.cuda.ExternalStream(sim.stream)
    a, b = cuda_events()
    sim.sync()
    a.record(s)
    for _ in range(steps):
        fn()
    b.record(s)
    b.synchronize()
    sim.sync()
    return a.elapsed_time(b)


def pin(arr: np.ndarray) -> bool:
    import torch
    rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
    return int(rc) == 0


def unpin(arr: np.ndarray):
    import torch
    torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except Exception:
        pass
    return 0


# --------------------------------------------------------------------------- sub-benchmarks (N=1)

def bench_propagate(lbm, warmup: int, reps: int, hbm_peak: float, layout: str = "soa", vl: int = 1) -> dict:
    """BASELINE config 1: 1024 x 8192 Philox input, repeated propagate prv -> nxt, 592 B/site."""
    lx, ly = 1024, 8192
    sim = lbm.Simulation(layout, lx, ly, vl, device=0)
    sim.init_philox(SEED)
    sim.bc("periodic")
    for _ in range(warmup):
        sim.propagate_only(sync=False)
    sim.set_profiling(True)
    sim.kernel_times()
    ms = time_steps(sim, reps, lambda: sim.propagate_only(sync=False))
    kt = sim.kernel_times()["propagate"]
    sim.set_profiling(False)
    t = kt[0] / kt[1] / 1e3
    gbs = lbm.propagate_gbps(lx, ly, 37, t, "nt")
    sim.close()
    return {"config": f"c1: 1024x8192 {layout}{vl if vl > 1 else ''}, Philox U[0,1) input, periodic halo, "
                      "propagate prv->nxt",
            "reps": reps, "ms_per_call": t * 1e3, "wall_ms_per_call": ms / reps, "GB_per_s": gbs,
            "frac_of_hbm": gbs / hbm_peak, "mlups": lbm.mlups(lx, ly, t)}


def bench_collide(lbm, warmup: int, reps: int, hbm_peak: float, layout: str = "soa", vl: int = 1) -> dict:
    """BASELINE config 2: 1024 x 8192 perturbed equilibrium, collide nxt -> prv, 1522 FLOP/site."""
    lx, ly = 1024, 8192
    sim = lbm.Simulation(layout, lx, ly, vl, device=0)
    sim.load(lbm.make_lattice("c2", lx, ly, SEED), which=1)
    for _ in range(warmup):
        sim.collide(1.0, sync=False)
    sim.set_profiling(True)
    sim.kernel_times()
    time_steps(sim, reps, lambda: sim.collide(1.0, sync=False))
    kt = sim.kernel_times()["collide"]
    sim.set_profiling(False)
    t = kt[0] / kt[1] / 1e3
    gf = lbm.collide_gflops(lx, ly, FLOPS_PER_SITE, t)
    gbs = lx * ly * BYTES_PER_SITE / t / 1e9
    sim.close()
    return {"config": f"c2: 1024x8192 {layout}{vl if vl > 1 else ''}, c2 perturbed equilibrium, collide nxt->prv, "
                      "omega 1.0",
            "reps": reps, "ms_per_call": t * 1e3, "GFLOP_per_s": gf, "mlups": lbm.mlups(lx, ly, t),
            "frac_of_fp64_nominal": gf / (FP64_NOMINAL_TFLOPS * 1e3), "GB_per_s": gbs,
            "frac_of_hbm": gbs / hbm_peak,
            "frac_of_attainable": gf / min(FP64_NOMINAL_TFLOPS * 1e3, FLOPS_PER_SITE / BYTES_PER_SITE * hbm_peak)}


def bench_config0(lbm, warmup: int) -> dict:
    """BASELINE config 0: 256 x 1024 RT init, wall bc, 100 full steps (one timed call of step(0.8, 100))."""
    lx, ly, n = 256, 1024, 100
    canon = lbm.make_lattice("rt", lx, ly, SEED)
    out = {}
    for layout, vl, variant in (("caosoa", 32, "fused"), ("soa", 1, "fused2"), ("soa", 1, "fused"),
                                ("soa", 1, "unfused")):
        sim = lbm.Simulation(layout, lx, ly, vl, device=0, bc="wall", variant=variant)
        sim.load(canon)
        sim.step(OMEGA, warmup)
        best = min(time_steps(sim, 1, lambda: sim.step(OMEGA, n, sync=False)) for _ in range(5))
        out[f"{layout}{vl if vl > 1 else ''}-{variant}"] = {"ms_per_100_steps": best,
                                                            "mlups": lx * ly * n / (best / 1e3) / 1e6}
        sim.close()
    return {"config": "c0: 256x1024, RT init, wall bc, omega 0.8, 100 steps per call (best of 5)", **out}


def bench_slab_schedule(lbm, layout, vl, ly, warmup, steps) -> dict:
    """The multi-GPU schedules on one GPU: a 1-rank NCCL ring (y-major columns through
    ncclSend/Recv to self) and a 1-rank P2P ring (the step kernel pushes its face columns into the
    ghost columns through peer memory, step counters in device memory) vs the plain single-domain
    step, same lattice.
    ly = 4096 is the per-GPU slab of the 8-GPU strong-scaling config (4096 x 32768 / 8)."""
    import torch  # noqa: F401  (NCCL comes from torch's libnccl.so.2)
    out = {}
    for name in ("single_domain", "nccl_self_ring", "p2p_self_ring"):
        if name == "single_domain":
            sim = lbm.Simulation(layout, LX, ly, vl, device=0, bc="periodic")
        elif name == "nccl_self_ring":
            sim = lbm.Simulation.slab(layout, LX, ly, vl, device=0, rank=0, nranks=1,
                                      nccl_id=lbm.nccl_unique_id(), bc="periodic")
        else:
            sim = lbm.Simulation.slab(layout, LX, ly, vl, device=0, rank=0, nranks=1, bc="periodic",
                                      transport="p2p")
        sim.init_rt_device(SEED)
        sim.step(OMEGA, warmup)
        sim.set_profiling(True)  # restarts the exposed-halo window (no warm-up exchanges)
        sim.set_profiling(False)
        ms = time_steps(sim, steps, lambda: sim.step(OMEGA, 1, sync=False))
        out[name] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6}
        if name != "single_domain":
            out[name]["exposed_halo_ms"] = sim.exposed_halo_ms()
        # per-kernel breakdown (separate, profiled pass)
        sim.set_profiling(True)
        sim.kernel_times()
        for _ in range(10):
            sim.step(OMEGA, 1, sync=False)
        kt = sim.kernel_times()
        sim.set_profiling(False)
        out[name]["kernel_ms_per_step"] = {k: v[0] / 10 for k, v in kt.items() if v[1]}
        out[name]["launches_per_step"] = {k: v[1] / 10 for k, v in kt.items() if v[1]}
        sim.close()
    out["schedule_overhead"] = out["nccl_self_ring"]["ms_per_step"] / out["single_domain"]["ms_per_step"] - 1.0
    out["p2p_schedule_overhead"] = out["p2p_self_ring"]["ms_per_step"] / out["single_domain"]["ms_per_step"] - 1.0
    out["config"] = (f"{LX}x{ly} {layout}{vl}, periodic y through NCCL to self / through the peer-memory "
                     f"push to self vs local wrap, {steps} steps")
    return out


def bench_slab_schedule_fused2(lbm, ly, warmup, steps) -> dict:
    """The FUSED2 y-slab schedule on one GPU: a 1-rank NCCL ring (6-row halos of both faces through
    ncclSend/Recv to self before every two-step sweep) vs the single domain, same lattice."""
    import torch  # noqa: F401  (NCCL comes from torch's libnccl.so.2)
    out = {}
    for name in ("single_domain", "nccl_self_ring"):
        if name == "single_domain":
            sim = lbm.Simulation("soa", LX, ly, 1, device=0, bc="periodic", variant="fused2")
        else:
            sim = lbm.Simulation.slab("soa", LX, ly, 1, device=0, rank=0, nranks=1, nccl_id=lbm.nccl_unique_id(),
                                      bc="periodic", variant="fused2")
        sim.init_rt_device(SEED)
        sim.step(OMEGA, warmup)
        sim.set_profiling(True)  # restarts the exposed-halo window (no warm-up exchanges) ...
        sim.set_profiling(False)  # ... without per-launch events in the timed loop
        ms = time_stepping(sim, steps, "fused2")
        out[name] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6}
        if name != "single_domain":
            out[name]["exposed_halo_ms_per_step"] = sim.exposed_halo_ms() / 2
        sim.close()
    out["schedule_overhead"] = out["nccl_self_ring"]["ms_per_step"] / out["single_domain"]["ms_per_step"] - 1.0
    out["config"] = (f"{LX}x{ly} soa FUSED2, periodic y through 6-row NCCL halos to self vs local wrap, "
                     f"{steps} steps")
    return out


def bench_fused2_group_emulation(lbm, nslabs, warmup, steps) -> dict:
    """BASELINE config 4 strong (4096 x 32768) as `nslabs` FUSED2 y-slabs on ONE GPU (group transport:
    6-row halos by device copies, each slab's sweep with its ghost-face bands), vs the same lattice
    as one domain: the cost of the decomposition at the per-GPU slab size of the 8-GPU run."""
    ly = STRONG_LY
    out = {"config": f"{LX}x{ly} soa FUSED2, walls, {nslabs} slabs on one GPU (device-copy halos) vs one domain, "
                     f"{steps} steps"}
    sim = lbm.Simulation("soa", LX, ly, 1, device=0, bc="wall", variant="fused2")
    sim.init_rt_device(SEED)
    sim.step(OMEGA, warmup)
    ms = time_stepping(sim, steps, "fused2")
    out["single_domain"] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6}
    sim.close()
    del sim
    grp = lbm.SlabGroup("soa", LX, ly, 1, nslabs, bc="wall", variant="fused2")
    for s in grp.slabs:  # the same global RT state, generated slab by slab on the device
        s.init_rt_device(SEED)
    grp.step(OMEGA, warmup)
    s0 = grp.slabs[0]
    ms = time_steps(s0, steps // 2, lambda: grp.step(OMEGA, 2))
    out[f"group_{nslabs}"] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6,
                             "timing": "CUDA events on the group's shared stream"}
    grp.close()
    out["decomposition_overhead"] = out[f"group_{nslabs}"]["ms_per_step"] / out["single_domain"]["ms_per_step"] - 1.0
    return out


def bench_p2p_ring_emulation(lbm, layout, vl, nslabs, warmup, steps) -> dict:
    """BASELINE config 4 strong (4096 x 32768) as `nslabs` P2P slabs on ONE GPU, stepped in
    lockstep through the real peer-memory protocol (counters, remote stores, separate streams),
    vs the same lattice as one domain.  The slabs share one GPU, so this measures the protocol's
    cost at the per-GPU slab size of the 8-GPU run, not NVLink."""
    import torch

    ly = STRONG_LY
    out = {"config": f"{LX}x{ly} {layout}{vl}, walls, {nslabs} P2P slabs on one GPU vs one domain, {steps} steps"}
    sim = lbm.Simulation(layout, LX, ly, vl, device=0, bc="wall")
    sim.init_rt_device(SEED)
    sim.step(OMEGA, warmup)
    ms = time_steps(sim, steps, lambda: sim.step(OMEGA, 1, sync=False))
    out["single_domain"] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6}
    sim.close()
    del sim
    slabs = lbm.p2p_ring(layout, LX, ly, vl, nslabs, bc="wall")
    for s in slabs:
        s.init_rt_device(SEED)
    lbm.step_slabs(slabs, OMEGA, warmup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lbm.step_slabs(slabs, OMEGA, steps)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0)
    out[f"p2p_ring_{nslabs}"] = {"ms_per_step": ms / steps, "mlups": LX * ly * steps / (ms / 1e3) / 1e6,
                                 "timing": "host wall clock around the lockstep loop (several streams)"}
    for s in slabs:
        s.close()
    out["protocol_overhead"] = out[f"p2p_ring_{nslabs}"]["ms_per_step"] / out["single_domain"]["ms_per_step"] - 1.0
    return out


def bench_variant(lbm, ly, layout, vl, variant, warmup, steps, hbm_peak: float = 0.0) -> dict:
    """BASELINE config 3: one step variant on 4096 x ly, with each kernel's roofline fraction
    (592 B/site per sweep against the HBM peak; collide also against the nominal FP64 peak)."""
    sim = lbm.Simulation(layout, LX, ly, vl, device=0, bc="wall", variant=variant)
    sim.init_rt_device(SEED)
    sim.step(OMEGA, warmup)
    sim.set_profiling(True)
    sim.kernel_times()
    ms = time_stepping(sim, steps, variant)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    sim.close()
    sites = LX * ly
    out = {"mlups": sites * steps / (ms / 1e3) / 1e6, "ms_per_step": ms / steps}
    for k, (tot, n) in kt.items():
        if n:
            kms = tot / n
            upd = steps_per_call(variant) if k == "fused" else 1  # time steps per launch
            out[f"{k}_ms"] = kms
            gbs = sites * BYTES_PER_SITE / (kms / 1e3) / 1e9  # one read + one write of the lattice per launch
            out[f"{k}_GBps"] = gbs
            if hbm_peak:
                out[f"{k}_frac_of_hbm"] = gbs / hbm_peak
            if k in ("fused", "collide"):
                out[f"{k}_frac_of_fp64_nominal"] = (upd * sites * FLOPS_PER_SITE / (kms / 1e3) /
                                                    (FP64_NOMINAL_TFLOPS * 1e12))
            if upd > 1:
                out[f"{k}_steps_per_launch"] = upd
    if variant == "fused2" and kt["fused"][1]:  # one launch per sweep
        sweep = kt["fused"][0] / kt["fused"][1]
        out["sweep_ms"] = sweep
        out["sweep_frac_of_hbm"] = sites * BYTES_PER_SITE / (sweep / 1e3) / 1e9 / hbm_peak if hbm_peak else None
    return out


# --------------------------------------------------------------------------- CPU baseline / reference arm

def physical_cores():
    """Physical cores of this host (psutil, else /proc/cpuinfo core ids), for the cpu_baseline record."""
    try:
        import psutil
        n = psutil.cpu_count(logical=False)
        if n:
            return int(n)
    except Exception:  # noqa: BLE001
        pass
    try:
        cores, phys = set(), None
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("physical id"):
                    phys = ln.split(":")[1].strip()
                elif ln.startswith("core id"):
                    cores.add((phys, ln.split(":")[1].strip()))
        return len(cores) or None
    except Exception:  # noqa: BLE001
        return None


def reference_step_rate(lx=LX, ly=1024, iterations=3, warmup=1, workers=None):
    """The unmodified reference step (oracle/_ref) on a bounded sample of the lattice."""
    from oracle import pyoracle as po
    workers = workers or os.cpu_count() or 1
    init = po.orc_lattice("rt", lx, ly, seed=SEED)
    sim = po.RefSim(po.AOS, lx, ly, 1, workers=workers)
    sim.load(init)
    med, _ = sim.time("step", omega=OMEGA, iterations=iterations, warmup=warmup)
    return lx * ly / med / 1e6, med, workers


def run_reference(args, dist):
    from oracle import pyoracle as po
    lx, ly = LX, 1024
    workers = os.cpu_count() or 1
    init = po.orc_lattice("rt", lx, ly, seed=SEED)
    sim = po.RefSim(po.AOS, lx, ly, 1, workers=workers)
    sim.load(init)
    for _ in range(args.warmup):
        sim.step(OMEGA, 1)
    t0 = time.perf_counter()
    times = []
    for _ in range(args.steps):
        a = time.perf_counter()
        sim.step(OMEGA, 1)
        times.append(time.perf_counter() - a)
    total = time.perf_counter() - t0
    value = lx * ly * args.steps / total / 1e6
    sample = (f"{lx}x{ly} rows of the {LX}x{LY_PER_GPU * args.gpus} lattice per step (RT init, "
              "reference step = periodic halo_exchange + propagate + collide; the reference has no wall bc), "
              "AoS layout (its fastest step here), ThreadPool of all host threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"c3/c4-weak sample: {lx}x{ly} (RT init, omega {OMEGA})", "lx": lx,
                       "ly_sample": ly, "layout": "aos", "workers": workers},
            "cpu_baseline": {"value": value, "unit": "MLUPS", "cores": workers, "kind": "reference",
                             "hardware_threads": os.cpu_count(), "physical_cores": physical_cores(),
                             "sample": sample},
            "e2e": {"value": value, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_ms_median": 1e3 * statistics.median(times)}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- main arm

def make_slab(lbm, args, dist: Dist, dev: int, ly_global: int):
    """This rank's slab: the peer-memory P2P transport (falls back to NCCL if the ranks cannot map
    each other's memory), or NCCL when asked."""
    rank, n = dist.rank, dist.world
    if args.transport == "p2p" and args.variant != "fused2":  # FUSED2 slabs exchange 6-row halos over NCCL
        sim, blob = None, b""
        try:
            sim = lbm.Simulation.slab(args.layout, LX, ly_global, args.vl, device=dev, rank=rank, nranks=n,
                                      bc="wall", variant=args.variant, transport="p2p")
            blob = sim.p2p_blob()
        except Exception as e:  # noqa: BLE001 -- reported, then NCCL
            print(f"[rank {rank}] p2p slab unavailable ({e}); using NCCL", file=sys.stderr, flush=True)
        ok = dist.min(1.0 if blob else 0.0) > 0.5
        if ok:  # every rank reaches the collectives below
            blobs = dist.all_gather_bytes(blob)
            try:
                sim.p2p_connect(blobs[(rank - 1) % n], blobs[(rank + 1) % n])
                conn = 1.0
            except Exception as e:  # noqa: BLE001
                print(f"[rank {rank}] p2p connect failed ({e}); using NCCL", file=sys.stderr, flush=True)
                conn = 0.0
            ok = dist.min(conn) > 0.5
        if ok:
            return sim, "p2p"
        if sim is not None:
            sim.close()
    uid0 = None
    if rank == 0:
        try:
            uid0 = lbm.nccl_unique_id()
        except Exception as e:  # noqa: BLE001 -- every rank learns it through the broadcast
            print(f"[rank 0] NCCL unavailable ({e})", file=sys.stderr, flush=True)
    uid = dist.bcast_bytes(uid0)
    if uid is None:
        if args.variant == "fused2":  # collectively: the single-sweep slabs with the peer-memory push
            print(f"[rank {rank}] FUSED2 slabs need NCCL; using the single-sweep CAoSoA32 P2P path",
                  file=sys.stderr, flush=True)
            args.layout, args.vl, args.variant, args.transport = "caosoa", 32, "fused", "p2p"
            return make_slab(lbm, args, dist, dev, ly_global)
        raise RuntimeError("no halo transport: P2P and NCCL both unavailable")
    sim = lbm.Simulation.slab(args.layout, LX, ly_global, args.vl, device=dev, rank=rank, nranks=n,
                              nccl_id=uid, bc="wall", variant=args.variant)
    return sim, "nccl"


def measure(lbm, args, dist: Dist, scaling: str) -> dict:
    """This rank's lattice for `scaling` (weak: --ly rows per GPU; strong: BASELINE config 4's
    4096 x 32768 split over the ranks), `--warmup` untimed steps, then exactly `--steps` timed
    steps between a barrier and a device sync on both sides; max over ranks."""
    n, dev = dist.world, dist.local
    ly_local = args.ly if scaling == "weak" else STRONG_LY // n
    ly_global = ly_local * n
    transport = None
    if n == 1:
        sim = lbm.Simulation(args.layout, LX, ly_local, args.vl, device=dev, bc="wall", variant=args.variant)
    else:
        sim, transport = make_slab(lbm, args, dist, dev, ly_global)
    sim.init_rt_device(SEED)  # each rank generates its slab of the global RT state on the device
    clocks = ClockSampler(dev)
    clocks.start()
    sim.step(OMEGA, args.warmup)
    sim.set_profiling(True)
    sim.kernel_times()
    dist.barrier()
    cuda_sync()
    ms = time_stepping(sim, args.steps, args.variant)
    cuda_sync()
    dist.barrier()
    kt = sim.kernel_times()
    sim.set_profiling(False)
    clk = clocks.stop()
    halo_ms = dist.max(sim.exposed_halo_ms()) if n > 1 else 0.0  # the slowest rank's exposed halo
    if n > 1 and args.variant == "fused2":
        halo_ms /= 2  # one 6-row exchange per two-step sweep
    ms_max = dist.max(ms)
    return {"sim": sim, "transport": transport, "ly_local": ly_local, "ly_global": ly_global, "ms_max": ms_max,
            "value": n * LX * ly_local * args.steps / (ms_max / 1e3) / 1e6, "kt": kt, "clk": clk,
            "halo_ms": halo_ms}


def single_gpu_rate(lbm, args, dist: Dist, ly: int):
    """Rank 0 alone, after the multi-GPU runs: the single-domain lattice of `ly` rows -- the 1-GPU
    point the N-GPU value is compared with (the other ranks wait at the barrier)."""
    val = None
    if dist.rank == 0:
        sim = lbm.Simulation(args.layout, LX, ly, args.vl, device=dist.local, bc="wall", variant=args.variant)
        sim.init_rt_device(SEED)
        sim.step(OMEGA, args.warmup)
        cuda_sync()
        ms = time_stepping(sim, args.steps, args.variant)
        cuda_sync()
        sim.close()
        val = LX * ly * args.steps / (ms / 1e3) / 1e6
    dist.barrier()
    return val


def run_b200(args, dist: Dist):
    if STUB:
        lbm = _StubLbm()
    else:
        import torch

        import paper_1804_01918_b200 as lbm
        torch.cuda.set_device(dist.local)
    dev = dist.local
    hbm_peak, peak_src = peaks()
    n = dist.world
    rank = dist.rank
    main = measure(lbm, args, dist, args.scaling)
    sim, transport, kt, clk = main["sim"], main["transport"], main["kt"], main["clk"]
    ly_local, ly_global, ms_max, value, halo_ms = (main["ly_local"], main["ly_global"], main["ms_max"],
                                                   main["value"], main["halo_ms"])
    sites_local = LX * ly_local
    launches = sum(c for _, c in kt.values())
    if transport == "p2p":  # + the one-thread step-counter wait and signal kernels of every step
        launches += 2 * args.steps

    fused_ms, fused_n = kt["fused"]
    dom = "fused" if fused_n else "collide"
    dom_ms = kt[dom][0] / max(1, kt[dom][1])
    form = None if STUB else lbm.set_fused2_tuning(-1, -1)[0]
    pair = args.variant == "fused2" and args.layout == "soa" and form == 4
    # single domain in the pair form: each timed "fused" interval is one k_step2_pair launch plus the
    # refresh of the images in the deep ghost rows for the next sweep (k_mirror6 at walls, k_wrap6 on
    # y-periodic domains; ~15 us, inside kernel_ms) -- two launches per sweep, as the ncu launch list shows
    if pair and not transport and not STUB:
        launches += fused_n
    # FUSED2: one sweep per timed "fused" interval (k_step2_pair + the face bands' k_step2_split beside it)
    # one launch reads and writes the lattice once (592 B/site) and advances `upd` time steps
    upd = steps_per_call(args.variant) if dom == "fused" else 1
    achieved = sites_local * BYTES_PER_SITE / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else None
    step_ms = ms_max / args.steps
    two = upd == 2
    roofline = {"bound": "hbm",
                "kernel": (("k_step2_pair_slab (y-slab sweep in the pair form: ghost-face bands first with the "
                            "6-row halo pack, interior in lockstep beside the NCCL exchange; two fused steps per "
                            "HBM sweep, two threads per site)" if pair and transport else
                            "k_step2_pair (two fused pull+collide steps per HBM sweep, temporal blocking; two "
                            "threads per site, 512-thread CTAs, lockstep band schedule; the walls as specular "
                            "images in the deep ghost rows, refreshed by k_mirror6 after the sweep)" if pair else
                            "k_step2_split (two fused pull+collide steps per HBM sweep, temporal blocking; "
                            "interior bands beside the two wall bands in one launch)") if two else
                           "k_collide<FAST,SHIFT> (fused pull-gather + collide)"),
                "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak if achieved else None,
                "traffic": load_ncu_traffic(args.layout, ly_local, args.variant, pair),
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": sites_local * BYTES_PER_SITE,
                "time_steps_per_launch": upd,
                "kernel_ms": dom_ms, "kernel_share_of_step": dom_ms / (step_ms * upd),
                "frac_of_nominal_hbm": achieved / HBM_NOMINAL_GBS if achieved else None,
                "nominal_hbm_gbs": HBM_NOMINAL_GBS,
                "fp64_tflops_reference_count": (upd * sites_local * FLOPS_PER_SITE / (dom_ms / 1e3) / 1e12
                                                if dom_ms > 0 else None),
                "frac_of_fp64_nominal": (upd * sites_local * FLOPS_PER_SITE / (dom_ms / 1e3) /
                                         (FP64_NOMINAL_TFLOPS * 1e12) if dom_ms > 0 else None),
                "edge_ms": kt["edge"][0] / max(1, kt["edge"][1])}
    if two:
        roofline["note"] = ("592 B/site per launch = per two time steps; the single-step bound at this "
                            "peak is peak/592 B site-steps/s, the two-step bound peak/296 B")

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e and not STUB:
        e2e = run_e2e(lbm, sim, args, dist)

    try:  # after the timed region: the FP64 denominator at the clocks this GPU holds under load
        fp64_meas = None if STUB else lbm.fp64_peak(dev)
    except Exception:  # noqa: BLE001
        fp64_meas = None
    if fp64_meas and roofline.get("fp64_tflops_reference_count"):
        roofline["fp64_peak_measured_tflops"] = fp64_meas
        roofline["frac_of_fp64_measured"] = roofline["fp64_tflops_reference_count"] / fp64_meas
    line = {"metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c3/c4-{args.scaling}: {LX}x{ly_local} per GPU (global {LX}x{ly_global}), RT init, "
                                   f"periodic x, top/bottom specular walls, omega {OMEGA}",
                       "lx": LX, "ly_per_gpu": ly_local, "ly_global": ly_global, "layout": args.layout,
                       "vl": args.vl if args.layout in ("csoa", "caosoa") else 1, "variant": args.variant,
                       "l2": "inputs larger than L2 (2 x 19.9 GB lattice per GPU vs 126 MB L2): no flush needed",
                       "parallelism": f"y-slab x{n}" if n > 1 else "single GPU",
                       "halo_transport": transport},
            "roofline": roofline, "gpu_launches": launches, "clocks": clk, "e2e": e2e,
            "exposed_halo_ms_per_step": halo_ms}
    if STUB:
        line["stub"] = "host-logic run: no-op lattice, host timers, gloo (not a measurement)"
    sim.close()
    del sim, main

    # ---- the other BASELINE config-4 scaling mode, same ranks (weak <-> strong)
    if not args.no_other_scaling:
        other = "strong" if args.scaling == "weak" else "weak"
        o = measure(lbm, args, dist, other)
        o["sim"].close()
        line[f"scaling_{other}"] = {
            "value": o["value"], "unit": "MLUPS", "n_gpus": n, "ms_per_step": o["ms_max"] / args.steps,
            "exposed_halo_ms_per_step": o["halo_ms"], "clocks": o["clk"], "halo_transport": o["transport"],
            "config": f"c4-{other}: {LX}x{o['ly_local']} per GPU (global {LX}x{o['ly_global']})"}
        del o
    # ---- the 1-GPU points (rank 0 alone), for the scaling efficiency of this run
    if n > 1 and not args.no_single:
        one_weak = single_gpu_rate(lbm, args, dist, args.ly)
        one_strong = single_gpu_rate(lbm, args, dist, STRONG_LY)
        ones = {"weak": one_weak, "strong": one_strong}
        line["single_gpu_mlups"] = ones
        if rank == 0:  # whole-job MLUPS / (N x the 1-GPU MLUPS of the same lattice per GPU / in total)
            eff = {args.scaling: value / (n * ones[args.scaling])}
            other = "strong" if args.scaling == "weak" else "weak"
            if f"scaling_{other}" in line:
                eff[other] = line[f"scaling_{other}"]["value"] / (n * ones[other])
            line["efficiency_vs_1gpu_same_run"] = eff

    if n == 1 and not args.no_extras and not STUB:
        kernels = {}
        for lay, vl in (("soa", 1), ("csoa", 32), ("caosoa", 32), ("aos", 1)):
            tag = f"{lay}{vl if vl > 1 else ''}"
            kernels[f"propagate_c1_{tag}"] = bench_propagate(lbm, 5, 200, hbm_peak, lay, vl)
            kernels[f"collide_c2_{tag}"] = bench_collide(lbm, 5, 200, hbm_peak, lay, vl)
        kernels["step_c0"] = bench_config0(lbm, 5)
        if fp64_meas:  # the collide-only kernels against the measured FP64 rate too
            for k, v in kernels.items():
                if k.startswith("collide_c2"):
                    v["frac_of_fp64_measured"] = v["GFLOP_per_s"] / (fp64_meas * 1e3)
            kernels["fp64_peak_measured_tflops"] = fp64_meas
        line["kernels"] = kernels
        # the other two BASELINE metrics, in the roofline record itself (propagate GB/s on config 1,
        # collide FP64 GFLOP/s on config 2 with the reference FLOP count), SoA and CAoSoA32
        roofline["propagate_c1"] = {
            tag: {"GB_per_s": kernels[f"propagate_c1_{tag}"]["GB_per_s"],
                  "frac_of_hbm": kernels[f"propagate_c1_{tag}"]["frac_of_hbm"], "unit": "GB/s",
                  "bytes_per_site": BYTES_PER_SITE}
            for tag in ("soa", "caosoa32")}
        roofline["collide_c2"] = {
            tag: {"GFLOP_per_s": kernels[f"collide_c2_{tag}"]["GFLOP_per_s"],
                  "frac_of_fp64_nominal": kernels[f"collide_c2_{tag}"]["frac_of_fp64_nominal"],
                  "frac_of_fp64_measured": kernels[f"collide_c2_{tag}"].get("frac_of_fp64_measured"),
                  "frac_of_attainable": kernels[f"collide_c2_{tag}"]["frac_of_attainable"],
                  "frac_of_hbm": kernels[f"collide_c2_{tag}"]["frac_of_hbm"],
                  "flop_per_site": FLOPS_PER_SITE, "unit": "GFLOP/s"}
            for tag in ("soa", "caosoa32")}
        variants = {}
        for lay, vl, var in (("soa", 1, "fused2"), ("soa", 1, "fused"), ("soa", 1, "unfused"), ("csoa", 32, "fused"),
                             ("csoa", 32, "unfused"), ("aos", 1, "fused"), ("caosoa", 32, "fused"),
                             ("caosoa", 32, "unfused")):
            if (lay, var) == (args.layout, args.variant):
                continue
            variants[f"{lay}{vl if vl > 1 else ''}-{var}"] = bench_variant(lbm, ly_local, lay, vl, var, 3, 20,
                                                                            hbm_peak)
        line["variants_c3"] = variants
        try:
            line["slab_schedule_fused2"] = {
                "strong_8gpu_slab": bench_slab_schedule_fused2(lbm, 4096, 4, 40),
                "weak_slab": bench_slab_schedule_fused2(lbm, LY_PER_GPU, 4, 20)}
        except Exception as e:  # noqa: BLE001
            line["slab_schedule_fused2"] = {"error": str(e)}
        try:
            line["fused2_group_emulation"] = bench_fused2_group_emulation(lbm, 8, 4, 20)
        except Exception as e:  # noqa: BLE001
            line["fused2_group_emulation"] = {"error": str(e)}
        # the single-step multi-GPU schedules (CAoSoA vl 32: NCCL columns / peer-memory push)
        try:
            line["slab_schedule"] = {
                "strong_8gpu_slab": bench_slab_schedule(lbm, "caosoa", 32, 4096, 3, 50),
                "weak_slab": bench_slab_schedule(lbm, "caosoa", 32, LY_PER_GPU, 3, 20)}
        except Exception as e:  # NCCL unavailable must not sink the line
            line["slab_schedule"] = {"error": str(e)}
        if args.p2p_extras:  # slabs on one GPU waiting on each other's counters: not on the default path
            try:
                line["p2p_ring_emulation"] = bench_p2p_ring_emulation(lbm, "caosoa", 32, 8, 3, 20)
            except Exception as e:  # noqa: BLE001
                line["p2p_ring_emulation"] = {"error": str(e)}
    if n == 1 and not args.no_cpu and not STUB:
        try:
            v, med, workers = reference_step_rate()
            line["cpu_baseline"] = {
                "value": v, "unit": "MLUPS", "cores": workers, "kind": "reference",
                "hardware_threads": os.cpu_count(), "physical_cores": physical_cores(),
                "sample": f"{LX}x1024 rows of the {LX}x{LY_PER_GPU} lattice, unmodified reference step "
                          f"(oracle/_ref, AoS, periodic halo_exchange + propagate + collide), median of 3 steps"}
        except Exception as e:  # the CPU baseline must not sink the GPU line
            line["cpu_baseline"] = {"value": None, "unit": "MLUPS", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_e2e(lbm, sim, args, dist: Dist):
    """Host canonical in -> n steps -> host canonical out through the public API, one pinned host
    canonical per rank.

    The rank's current state is dumped into the host buffer first.  The headline call is the streamed
    run, Simulation.run(host, omega, n, out=host) (d2q37_run_canonical): on a single wall domain the
    upload, the sweeps and the download are pipelined in y-chunks, bit-identical to the three verbs.
    The three verbs one after another (load + step + dump: nothing overlaps) are timed beside it.
    Slab ranks have no streamed path and time the three verbs only.
    """
    nsteps = args.e2e_steps
    need = 37 * sim.lx * sim.ly * 8
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", dist.world))
    avail = host_mem_available()
    enough = not (avail and avail < need * local_ranks * 1.25)
    if dist.min(1.0 if enough else 0.0) < 0.5:  # collective: every rank steps, or none does
        return {"value": None, "unit": "MLUPS",
                "skipped": f"{local_ranks} x {need / 1e9:.1f} GB host buffers exceed available host memory"}
    canon = np.empty((37, sim.lx, sim.ly), dtype=np.float64)
    pinned = pin(canon)
    sim.dump(out=canon)
    sites = LX * sim.ly * dist.world

    def three_verbs():
        sim.load(canon)
        sim.step(OMEGA, nsteps)
        sim.dump(out=canon)

    def streamed():
        sim.run(canon, OMEGA, nsteps, out=canon)

    def timed(call):
        times = []
        for _ in range(1 + args.e2e_iters):  # first call warms the pinned path
            dist.barrier()
            t0 = time.perf_counter()
            call()
            times.append(time.perf_counter() - t0)
        return dist.max(min(times[1:]))

    t3 = timed(three_verbs)
    rec = {"unit": "MLUPS", "h2d_bytes_per_step": need / nsteps, "d2h_bytes_per_step": need / nsteps,
           "steps_per_call": nsteps, "h2d_bytes_per_call": need, "d2h_bytes_per_call": need, "pinned": pinned,
           "three_verbs": {"value": sites * nsteps / t3 / 1e6, "seconds_per_call": t3,
                           "call": f"Simulation.load(host canonical) + step(0.8, n, {sim.variant}, wall) + "
                                   "dump(host canonical)"}}
    if dist.world == 1 and sim.variant == "fused2":
        t = timed(streamed)
        rec.update({"value": sites * nsteps / t / 1e6, "seconds_per_call": t,
                    "call": f"Simulation.run(host canonical, 0.8, n, out=host canonical) [{sim.variant}, wall]: "
                            "upload, sweeps and download pipelined in y-chunks (d2q37_run_canonical)"})
    else:
        rec.update({"value": rec["three_verbs"]["value"], "seconds_per_call": t3,
                    "call": rec["three_verbs"]["call"]})
    if pinned:
        unpin(canon)
    return rec


def load_ncu_traffic(layout: str, ly: int, variant: str = "fused", pair: bool = False):
    """DRAM bytes/launch of the step kernel from the committed ncu capture (profiles/), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_fused_traffic.json")
    key = {"csoa": "prof_fused_csoa", "caosoa": "prof_fused_caosoa"}.get(layout, "prof_fused")
    if variant == "fused2" and layout == "soa":
        key = "prof_step2_pair" if pair else "prof_step2_soa"
    try:
        with open(path) as f:
            rec = json.load(f)[key]
    except Exception:
        return None
    # the capture is of the 4096 x 16384 launch; scale per site for other slab heights
    return rec["dram_bytes_per_launch"] * (LX * ly) / (4096 * 16384)


def launch_ranks(args):
    """`--gpus N` without a launcher: start N ranks (one per GPU) through torch.distributed.run on
    127.0.0.1 and exit with their status.  Fails loudly -- never a silent 1-GPU line -- when this
    host has fewer than N GPUs."""
    import socket
    if not STUB:
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            have = 0
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but this host has {have} CUDA device(s)")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--layout", choices=["aos", "soa", "csoa", "caosoa"], default=None,
                    help="default: soa (the FUSED2 store)")
    ap.add_argument("--vl", type=int, default=None)
    ap.add_argument("--variant", choices=["fused", "unfused", "fused2"], default=None,
                    help="default: fused2 (two steps per HBM sweep)")
    ap.add_argument("--ly", type=int, default=LY_PER_GPU, help="rows per GPU (weak scaling)")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 halo transport: peer-memory push from the step kernel, or NCCL")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: --ly rows per GPU; strong: 4096 x 32768 split over the GPUs (config 4)")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--e2e-iters", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-other-scaling", action="store_true",
                    help="skip the second config-4 measurement (strong when --scaling weak and vice versa)")
    ap.add_argument("--no-single", action="store_true", help="N > 1: skip the 1-GPU points of the efficiency")
    ap.add_argument("--p2p-extras", action="store_true",
                    help="also run the 8-slab P2P ring emulation on one GPU (slabs spin on each other)")
    ap.add_argument("--stub", action="store_true",
                    help="host-logic test mode: no-op lattice, host timers, gloo (tests/test_bench_launch.py)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)  # timing rule: at least 3 warm-up steps
    multi = int(os.environ.get("WORLD_SIZE", "1")) > 1
    if args.layout is None:
        args.layout = "soa"
    if args.vl is None:
        args.vl = 32 if args.layout in ("csoa", "caosoa") else 1
    if args.variant is None:
        args.variant = "fused2"
    del multi
    global STUB
    STUB = args.stub
    if args.impl == "reference":
        # rank 0 alone runs the CPU reference; other ranks exit 0 without work
        if int(os.environ.get("RANK", "0")) == 0:
            run_reference(args, None)
        return
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        launch_ranks(args)  # re-executes this script as args.gpus ranks; does not return
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mismatched run")
    dist = Dist()
    try:
        run_b200(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
