"""FUSED2 on the banded store vs the SoA store on the bench lattice (alternated A/B/A/B).
Usage: python tools/fused2_banded_time.py [lx ly] (BC=wall|periodic)"""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 16384)))
BC = os.environ.get("BC", "wall")
n = 20
res = {}
for rep in range(2):
    for layout in ("soa", "banded"):
        s = lbm.Simulation(layout, lx, ly, 1, device=0, bc=BC, variant="fused2")
        s.init_rt_device(12345)
        s.step(0.8, 4)
        s.sync()
        best = 1e9
        for _ in range(2):
            t0 = time.perf_counter()
            s.step(0.8, n)
            s.sync()
            best = min(best, time.perf_counter() - t0)
        s.set_profiling(True)
        s.step(0.8, 4)
        kt = s.kernel_times()["fused"]
        s.close()
        res.setdefault(layout, []).append(best)
        print(f"{lx}x{ly} {BC} {layout:7s}: {best / n * 1e3:.3f} ms/step = {lx * ly * n / best / 1e6:.0f} MLUPS"
              f"  sweep kernel {kt[0] / max(1, kt[1]):.3f} ms", flush=True)
