"""run_validation on the GPU (validation.hpp:44-92, validation.cpp:73-123).

Every (geometry, layout, vl) case loads the same seeded random lattice, runs
the reference's unfused verbs on the device -- ``halo_exchange`` (bc periodic),
``propagate`` with the (optionally corrupted) offset table, ``collide`` -- for
``steps`` steps, and compares the canonical dump bit for bit against the
scalar device reference (:func:`paper_1804_01918_b200.scalar_steps`: a
halo-free canonical array with explicit modulo indexing and the same collide
arithmetic).  The first diverging (x, y, p) in the reference's loop order is
reported, and ``print_report`` writes the reference's report lines.
"""
from __future__ import annotations

import dataclasses
import sys

import numpy as np

from . import make_lattice, scalar_steps, Simulation

__all__ = ["ValidationOptions", "Divergence", "CaseResult", "ValidationReport", "run_validation", "print_report"]


@dataclasses.dataclass
class ValidationOptions:
    """ValidationOptions (validation.hpp:44-58); ``workers``/``schedule`` are accepted and
    ignored (the CUDA grid replaces the pool); ``math`` picks the collide arithmetic of both
    sides; ``device`` the GPU."""
    geometries: list = dataclasses.field(default_factory=lambda: [(16, 32), (64, 128)])
    vls: list = dataclasses.field(default_factory=lambda: [1, 2, 4, 8])
    layouts: list = dataclasses.field(default_factory=lambda: ["aos", "soa", "csoa", "caosoa"])
    steps: int = 10
    omega: float = 1.0
    seed: int = 12345
    workers: int = 4
    schedule: str = "dynamic"
    corrupt_population: int = -1
    math: str = "fast"
    device: int = 0


@dataclasses.dataclass
class Divergence:
    x: int
    y: int
    p: int
    got: float
    want: float


@dataclasses.dataclass
class CaseResult:
    lx: int
    ly: int
    layout: str
    vl: int
    passed: bool
    divergence: Divergence | None = None


@dataclasses.dataclass
class ValidationReport:
    cases: list
    passed: bool


def first_divergence(got: np.ndarray, want: np.ndarray) -> Divergence | None:
    """First (x, y, p) in x-then-y-then-p order whose bits differ (validation.cpp:59-70)."""
    diff = got.view(np.uint64) != want.view(np.uint64)  # (37, lx, ly)
    if not diff.any():
        return None
    order = np.transpose(diff, (1, 2, 0)).reshape(-1)  # x, y, p
    i = int(np.argmax(order))
    npop, _, ly = diff.shape
    x, rem = divmod(i, ly * npop)
    y, p = divmod(rem, npop)
    return Divergence(x, y, p, float(got[p, x, y]), float(want[p, x, y]))


def run_validation(opts: ValidationOptions | None = None) -> ValidationReport:
    opts = opts or ValidationOptions()
    if opts.schedule not in ("dynamic", "static"):
        raise ValueError(f"unknown schedule: {opts.schedule}")
    if opts.workers < 1:
        raise ValueError("worker count must be >= 1")
    cases = []
    for lx, ly in opts.geometries:
        seed = (opts.seed ^ ((lx << 32) | ly)) & 0xFFFFFFFFFFFFFFFF
        initial = make_lattice("random", lx, ly, seed)
        want = scalar_steps(initial, opts.omega, opts.steps, math=opts.math, device=opts.device)
        for layout in opts.layouts:
            for vl in opts.vls:
                sim = Simulation(layout, lx, ly, vl, device=opts.device, math=opts.math)
                try:
                    sim.load(initial)
                    for _ in range(opts.steps):
                        sim.bc("periodic", sync=False)
                        sim.propagate_only(opts.corrupt_population, sync=False)
                        sim.collide(opts.omega, sync=False)
                    sim.sync()
                    d = first_divergence(sim.dump(), want)
                finally:
                    sim.close()
                cases.append(CaseResult(lx, ly, layout, vl, d is None, d))
    return ValidationReport(cases, all(c.passed for c in cases))


def print_report(report: ValidationReport, file=None) -> None:
    """print_report (validation.cpp:125-139): one line per case and a summary line."""
    out = file or sys.stdout
    for c in report.cases:
        line = f"{'pass' if c.passed else 'FAIL'}  {c.lx}x{c.ly}  {c.layout}  vl={c.vl}"
        if c.divergence:
            d = c.divergence
            line += f"  first divergence at (x={d.x}, y={d.y}, p={d.p}): got {d.got:.6g}, want {d.want:.6g}"
        print(line, file=out)
    print(f"validation {'passed' if report.passed else 'FAILED'} ({len(report.cases)} cases)", file=out)


def main(argv=None) -> int:
    """``python -m paper_1804_01918_b200.validation`` -- the device analogue of ``lbmbench
    validate`` (lbmbench_main.cpp:102-125): bare, it runs the default suite (both stock
    geometries, vl 1/2/4/8); exit status 0 iff every case passes."""
    import argparse

    ap = argparse.ArgumentParser(description=main.__doc__.splitlines()[0])
    ap.add_argument("--lx", type=int)
    ap.add_argument("--ly", type=int)
    ap.add_argument("--vl", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--layout", nargs="+", default=["aos", "soa", "csoa", "caosoa"],
                    choices=["aos", "soa", "csoa", "caosoa"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--omega", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--math", choices=["fast", "strict"], default="fast")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--corrupt-population", type=int, default=-1)
    ap.add_argument("-o", "--output", help="write the report here instead of stdout")
    a = ap.parse_args(argv)
    opts = ValidationOptions(vls=a.vl, layouts=a.layout, steps=a.steps, omega=a.omega, seed=a.seed, math=a.math,
                             device=a.device, corrupt_population=a.corrupt_population)
    if a.lx is not None or a.ly is not None:
        opts.geometries = [(a.lx or 16, a.ly or 32)]
    rep = run_validation(opts)
    if a.output:
        with open(a.output, "w") as f:
            print_report(rep, f)
    else:
        print_report(rep)
    return 0 if rep.passed else 1


if __name__ == "__main__":
    sys.exit(main())
