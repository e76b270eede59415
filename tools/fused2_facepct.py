"""FUSED2 face-band CTA share sweep (d2q37_set_fused2_tuning face_pct) for one form: python tools/fused2_facepct.py FORM lx ly bc pct..."""
import sys
import time

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

form, lx, ly, bc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
n = 40
for pct in (int(a) for a in sys.argv[5:]):
    lbm.set_fused2_tuning(form, pct)
    s = lbm.Simulation("soa", lx, ly, 1, device=0, bc=bc, variant="fused2")
    s.init_rt_device(12345)
    s.step(0.8, 6)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        s.step(0.8, n)
        best = min(best, time.perf_counter() - t0)
    s.close()
    print(f"form {form} {lx}x{ly} {bc} face_pct {pct}: {best / n * 1e3:.3f} ms/step = {lx * ly * n / best / 1e6:.0f} MLUPS",
          flush=True)
