"""Times FUSED2 (two steps per sweep, SoA) against FUSED (CAoSoA32 / SoA) on the bench lattice."""
import sys
import time

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 16384)))
n = 40
import os
BC = os.environ.get("BC", "wall")
ONLY = os.environ.get("ONLY")
for layout, vl, variant in (("caosoa", 32, "fused"), ("soa", 1, "fused"), ("soa", 1, "fused2")):
    if ONLY and variant != ONLY:
        continue
    s = lbm.Simulation(layout, lx, ly, vl, device=0, bc=BC, variant=variant)
    s.init_rt_device(12345)
    s.step(0.8, 4)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        s.step(0.8, n)
        best = min(best, time.perf_counter() - t0)
    s.set_profiling(True)
    s.step(0.8, 4)
    kt = s.kernel_times()
    s.close()
    print(f"{layout:7s} vl {vl:2d} {variant:7s}: {best / n * 1e3:.3f} ms/step = {lx * ly * n / best / 1e6:.0f} MLUPS  kernels {kt}",
          flush=True)
