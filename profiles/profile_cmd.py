#!/usr/bin/env python3
"""Small, ncu-friendly drivers of the three hot kernels (the commands the profiles/ captures come from).

  --case step       4096x16384 SoA, RT init, wall bc, omega 0.8, fused steps   (bench workload)
  --case unfused    same lattice, unfused steps (edge + propagate + collide)
  --case csoa       same lattice, CSoA vl=32 fused steps
  --case caosoa     same lattice, CAoSoA vl=32 fused steps                    (bench default)
  --case propagate  1024x8192 Philox input, propagate prv->nxt (--layout/--vl, default SoA)  (BASELINE config 1)
  --case collide    1024x8192 c2 input, collide nxt->prv (--layout/--vl, default SoA)         (BASELINE config 2)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1804_01918_b200 as lbm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="step", choices=["step", "unfused", "csoa", "caosoa", "propagate", "collide"])
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--lx", type=int, default=4096)
    ap.add_argument("--ly", type=int, default=16384)
    ap.add_argument("--layout", default="soa", help="propagate / collide cases: layout (soa, csoa, caosoa, aos)")
    ap.add_argument("--vl", type=int, default=1)
    a = ap.parse_args()
    if a.case in ("step", "unfused", "csoa", "caosoa"):
        layout, vl = (a.case, 32) if a.case in ("csoa", "caosoa") else ("soa", 1)
        s = lbm.Simulation(layout, a.lx, a.ly, vl, bc="wall", variant="unfused" if a.case == "unfused" else "fused")
        s.load(lbm.make_lattice("rt", a.lx, a.ly, 12345))
        for _ in range(a.steps):
            s.step(0.8, 1, sync=False)
        s.sync()
    elif a.case == "propagate":
        s = lbm.Simulation(a.layout, 1024, 8192, a.vl)
        s.init_philox(12345)
        s.bc("periodic")
        for _ in range(a.steps):
            s.propagate_only(sync=False)
        s.sync()
    else:
        s = lbm.Simulation(a.layout, 1024, 8192, a.vl)
        s.load(lbm.make_lattice("c2", 1024, 8192, 12345), which=1)
        for _ in range(a.steps):
            s.collide(1.0, sync=False)
        s.sync()
    print(f"{a.case}: ok, {s.time_step} steps")


if __name__ == "__main__":
    main()
