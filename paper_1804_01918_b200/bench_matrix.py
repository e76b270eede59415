"""GPU rows in the reference's benchmark CSV (schema v1), with NVML energy.

Mirror of ``run_bench_matrix`` (proj/src/bench_matrix.cpp:34-115),
``time_kernel`` / ``finalize_metrics`` / ``write_csv_*`` (metrics.cpp:73-122)
and the energy columns (energy.cpp:88-118) for the device lattice:

* one row per (kernel in propagate/collide/step, layout, vl) cell, shear init
  (``make_shear_lattice(amp 0.02, t0)``, bench_matrix.cpp:57), one periodic
  halo exchange before timing (:79);
* ``t_iter_s`` / ``t_min_s`` = median / min of per-iteration CUDA-event times
  after ``warmup`` untimed calls; derived columns recompute exactly from the
  row (acceptance C7);
* ``workers`` = GPUs (1); ``traffic_model`` = nt (the device writes whole
  sectors, no read-for-ownership); ``clock_res_ns`` = CUDA event resolution;
* energy: NVML board energy (``nvmlDeviceGetTotalEnergyConsumption``) in the
  package column, the DRAM column empty (no counter); rows without a usable
  NVML get no energy columns, like a host without powercap (acceptance C8);
* a cell whose geometry is rejected is recorded with ``status = error: ...``
  and the run continues (bench_matrix.cpp:59-72).

Usage (mirrors ``lbmbench bench``)::

    python -m paper_1804_01918_b200.bench_matrix --lx 1024 --ly 8192 --vl 32 \\
        --iterations 50 --warmup 5 --energy -o bench.csv
"""
from __future__ import annotations

import argparse
import statistics
import sys
from dataclasses import dataclass, field

import paper_1804_01918_b200 as lbm

CSV_SCHEMA_VERSION = 1
CUDA_EVENT_RESOLUTION_NS = 500.0  # cudaEventElapsedTime resolution (~0.5 us)
LAYOUTS = ("aos", "soa", "csoa", "caosoa")
KERNELS = ("propagate", "collide", "step")


@dataclass
class BenchReport:
    kernel: str
    layout: str
    vl: int
    workers: int
    lx: int
    ly: int
    iterations: int
    warmup: int
    traffic: str = "nt"
    flops_per_site: float = float(lbm.COLLIDE_FLOPS_PER_SITE)
    t_iter_s: float = 0.0
    t_min_s: float = 0.0
    mlups: float = 0.0
    gbps: float = 0.0
    gflops: float = 0.0
    clock_res_ns: float = CUDA_EVENT_RESOLUTION_NS
    energy: dict | None = None
    status: str = "ok"
    samples_s: list = field(default_factory=list)


def sweeps_of(kernel: str) -> int:
    """metrics.cpp:90: a full step moves every element twice."""
    return 2 if kernel == "step" else 1


def finalize_metrics(r: BenchReport) -> None:
    """metrics.cpp:92-98."""
    r.mlups = lbm.mlups(r.lx, r.ly, r.t_iter_s)
    r.gbps = lbm.propagate_gbps(r.lx, r.ly, lbm.NPOP, r.t_iter_s, r.traffic) * sweeps_of(r.kernel)
    r.gflops = 0.0 if r.kernel == "propagate" else lbm.collide_gflops(r.lx, r.ly, r.flops_per_site, r.t_iter_s)


def _fmt6(v: float) -> str:
    return "%.6g" % v


def write_csv_header(out, energy_columns: bool) -> None:
    """metrics.cpp:100-106."""
    out.write("schema_version,kernel,layout,vl,workers,lx,ly,iterations,warmup,traffic_model,"
              "flops_per_site,t_iter_s,t_min_s,mlups,gbps,gflops,clock_res_ns")
    if energy_columns:
        out.write(",energy_pkg_j,energy_dram_j,energy_total_j,avg_power_w")
    out.write(",status\n")


def write_csv_row(out, r: BenchReport, energy_columns: bool) -> None:
    """metrics.cpp:108-122."""
    cols = [str(CSV_SCHEMA_VERSION), r.kernel, r.layout, str(r.vl), str(r.workers), str(r.lx), str(r.ly),
            str(r.iterations), str(r.warmup), r.traffic, _fmt6(r.flops_per_site), _fmt6(r.t_iter_s),
            _fmt6(r.t_min_s), _fmt6(r.mlups), _fmt6(r.gbps), _fmt6(r.gflops), _fmt6(r.clock_res_ns)]
    if energy_columns:
        if r.energy:
            e = r.energy
            cols += [_fmt6(e["joules_package"]), "", _fmt6(e["joules_total"]), _fmt6(e["avg_power_w"])]
        else:
            cols += ["", "", "", ""]
    cols.append(r.status)
    out.write(",".join(cols) + "\n")


class NvmlEnergy:
    """RAPL analogue: cumulative board energy of one GPU (mJ, 64-bit, no wrap)."""

    def __init__(self, device: int = 0):
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            pynvml.nvmlDeviceGetTotalEnergyConsumption(self._h)
            self.ok = True
        except Exception:
            self.ok = False

    def read_mj(self) -> int:
        return int(self._nvml.nvmlDeviceGetTotalEnergyConsumption(self._h))


def time_kernel(sim, body, iterations: int, warmup: int):
    """metrics.cpp:73-88 with CUDA events on the lattice stream instead of steady_clock."""
    import torch

    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    for _ in range(warmup):
        body()
    sim.sync()
    stream = torch.cuda.ExternalStream(sim.stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iterations)]
    for a, b in evs:
        a.record(stream)
        body()
        b.record(stream)
    evs[-1][1].synchronize()
    sim.sync()
    samples = [a.elapsed_time(b) / 1e3 for a, b in evs]
    return statistics.median(samples), min(samples), samples


def energy_per_iteration(sim, body, provider: NvmlEnergy, t_iter_s: float, window_s: float = 1.0) -> dict:
    """Joules per call over a window of >= window_s: the NVML energy counter updates
    every few tens of ms, so the timed iterations alone are too short to read it."""
    import time

    reps = max(1, int(window_s / max(t_iter_s, 1e-6)))
    sim.sync()
    before, t0 = provider.read_mj(), time.perf_counter()
    for _ in range(reps):
        body()
    sim.sync()
    wall = time.perf_counter() - t0
    joules = (provider.read_mj() - before) / 1e3 / reps
    return {"joules_package": joules, "joules_total": joules, "avg_power_w": joules * reps / wall,
            "window_s": wall, "calls": reps}


def run_bench_matrix(lx: int, ly: int, layouts=LAYOUTS, vls=(8,), iterations: int = 50, warmup: int = 5,
                     omega: float = 1.0, energy: bool = False, csv=sys.stdout, log=sys.stderr, device: int = 0):
    """bench_matrix.cpp:34-115 for the device lattice; returns the BenchReports."""
    provider = NvmlEnergy(device) if energy else None
    energy_columns = bool(provider and provider.ok)
    if energy and not energy_columns:
        log.write("energy counters unavailable on this host; energy columns omitted\n")
    write_csv_header(csv, energy_columns)
    reports = []
    model = lbm.model()
    for layout in layouts:
        for vl in vls:
            rows = [BenchReport(k, layout, vl, 1, lx, ly, iterations, warmup) for k in KERNELS]
            try:
                sim = lbm.Simulation(layout, lx, ly, vl, device=device, bc="periodic", variant="fused")
                sim.init_shear(0.02, model.t0)
                sim.bc("periodic")
            except Exception as e:  # the whole cell is unusable: record it and move on
                for r in rows:
                    r.status = f"error: {e}"
                    write_csv_row(csv, r, energy_columns)
                    reports.append(r)
                continue
            bodies = {
                "propagate": lambda: sim.propagate_only(sync=False),
                "collide": lambda: sim.collide(omega, sync=False),
                "step": lambda: sim.step(omega, 1, sync=False),
            }
            for r in rows:
                try:
                    # warm up before the energy window (bench_matrix.cpp:88-91)
                    for _ in range(warmup):
                        bodies[r.kernel]()
                    sim.sync()
                    r.t_iter_s, r.t_min_s, r.samples_s = time_kernel(sim, bodies[r.kernel], iterations, 0)
                    if energy_columns:
                        r.energy = energy_per_iteration(sim, bodies[r.kernel], provider, r.t_iter_s)
                    finalize_metrics(r)
                except Exception as e:
                    r.status = f"error: {e}"
                write_csv_row(csv, r, energy_columns)
                reports.append(r)
            sim.close()
    return reports


def write_trend_summary(out, reports) -> None:
    """bench_matrix.cpp:117-142."""
    prop, coll = {}, {}
    for r in reports:
        if r.status != "ok":
            continue
        if r.kernel == "propagate":
            prop.setdefault(r.layout, []).append(r.gbps)
        if r.kernel == "collide":
            coll.setdefault(r.layout, []).append(r.mlups)
    if not prop and not coll:
        return
    out.write("device trend summary (best over the matrix):\n")
    for layout, v in prop.items():
        out.write(f"  propagate {layout}: {max(v):g} GB/s\n")
    for layout, v in coll.items():
        out.write(f"  collide   {layout}: {max(v):g} MLUPS\n")
    if "csoa" in prop and "aos" in prop:
        out.write(f"  propagate csoa/aos bandwidth ratio: {max(prop['csoa']) / max(prop['aos']):g}\n")
    if "caosoa" in coll and "soa" in coll:
        out.write(f"  collide caosoa/soa throughput ratio: {max(coll['caosoa']) / max(coll['soa']):g}\n")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="D2Q37 device bench matrix (reference CSV schema v1)")
    ap.add_argument("--lx", type=int, default=256)
    ap.add_argument("--ly", type=int, default=1024)
    ap.add_argument("--layouts", default=",".join(LAYOUTS))
    ap.add_argument("--vl", default="8")
    ap.add_argument("--iterations", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--omega", type=float, default=1.0)
    ap.add_argument("--energy", action="store_true")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("-o", "--output", default="")
    a = ap.parse_args(argv)
    out = open(a.output, "w") if a.output else sys.stdout
    try:
        reports = run_bench_matrix(a.lx, a.ly, a.layouts.split(","), [int(v) for v in a.vl.split(",")],
                                   a.iterations, a.warmup, a.omega, a.energy, out, sys.stderr, a.device)
    finally:
        if a.output:
            out.close()
    write_trend_summary(sys.stderr, reports)
    return 0


if __name__ == "__main__":
    sys.exit(main())
