"""Times the overlapped FUSED2 slab sweep kernels through the test hook (no exchange) per face pair:
python tools/slab_sweep_time.py [lx ly]  -- pair form (4) and one-thread form (0), ghost/ghost, wall/ghost."""
import sys
import time

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (2048, 16384)))
init = lbm.make_lattice("random", lx, ly, seed=5)  # finite deep ghost rows are zero: keep rho well above 0
for faces in (("ghost", "ghost"), ("wall", "ghost"), ("ghost", "wall")):
    for form in (4, 0):
        s = lbm.Simulation("soa", lx, ly, 1, device=0, bc="wall", variant="fused2")
        best = 1e9
        for _ in range(4):  # one sweep per load: zero ghost rows drain mass near the faces over many sweeps
            s.load(init)
            s.sync()
            t0 = time.perf_counter()
            s.debug_step2_slab_sweep(0.8, form, *faces)
            best = min(best, time.perf_counter() - t0)
        n = 1
        s.close()
        print(f"{lx}x{ly} faces {faces[0]}/{faces[1]} form {form}: {best / n * 1e3:.3f} ms/sweep = "
              f"{2 * lx * ly * n / best / 1e6:.0f} MLUPS", flush=True)
