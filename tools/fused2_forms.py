"""FUSED2 interior-band forms on the bench lattice: per-thread loads (0) vs bulk-copy staging (1).

Alternates the forms (A/B/A/B) on one lattice so clock drift cancels; checks they are bit-identical.
Usage: python tools/fused2_forms.py [lx ly] (BC=wall|periodic, FACE=<pct>)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 16384)))
BC = os.environ.get("BC", "wall")
FACE = int(os.environ.get("FACE", "0"))
n = 20
FORMS = [int(f) for f in os.environ.get("FORMS", "0 1").split()]
s = lbm.Simulation("soa", lx, ly, 1, device=0, bc=BC, variant="fused2")
s.init_rt_device(12345)
res = {f: [] for f in FORMS}
for rep in range(3):
    for form in FORMS:
        lbm.set_fused2_tuning(form, FACE)
        s.step(0.8, 4)
        s.sync()
        t0 = time.perf_counter()
        s.step(0.8, n)
        s.sync()
        res[form].append(time.perf_counter() - t0)
for form in FORMS:
    best = min(res[form])
    print(f"{lx}x{ly} {BC} form {form}: {best / n * 1e3:.3f} ms/step = {lx * ly * n / best / 1e6:.0f} MLUPS "
          f"(all: {[round(lx * ly * n / t / 1e6) for t in res[form]]})", flush=True)
s.set_profiling(True)
for form in FORMS:
    lbm.set_fused2_tuning(form, FACE)
    s.step(0.8, 4)
    print("form", form, "kernel times", s.kernel_times(), flush=True)
s.close()
# bit-identity of the two forms (split-launch size, host copies kept small)
outs = []
for form in FORMS:
    lbm.set_fused2_tuning(form, FACE)
    t = lbm.Simulation("soa", lx, min(ly, 2048), 1, device=0, bc=BC, variant="fused2")
    t.init_rt_device(777)
    t.step(0.8, 4)
    outs.append(t.dump())
    t.close()
print("forms bit-identical:", all(np.array_equal(outs[0], o) for o in outs), flush=True)
