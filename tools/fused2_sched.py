"""FUSED2 interior (form, schedule) A/B: forms 0-3 (d2q37_set_fused2_tuning), schedules band-major (0) /
lockstep (1).

Times FUSED2 sweeps (SoA, RT init) per variant on a few lattices and checks
that every variant leaves a bit-identical state (hash of the dumped canonical
state on the small lattices, of the moments on the large ones).
Usage: VARIANTS="0:0 0:1 3:1" python tools/fused2_sched.py [lx ly bc] ...   (default: the bench set)
"""
import os
import hashlib
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1804_01918_b200 as lbm  # noqa: E402

cases = [(4096, 16384, "wall"), (4096, 32768, "wall"), (4096, 16384, "periodic"), (4096, 8192, "wall"),
         (4096, 4096, "wall"), (4096, 2048, "wall")]
if len(sys.argv) > 3:
    a = sys.argv[1:]
    cases = [(int(a[i]), int(a[i + 1]), a[i + 2]) for i in range(0, len(a) - 2, 3)]
n = 40
for lx, ly, bc in cases:
    res = {}
    for var in os.environ.get("VARIANTS", "0:0 0:1").split():
        form, sched = (int(v) for v in var.split(":"))
        lbm.set_fused2_tuning(form, -1)
        lbm.set_fused2_schedule(sched)
        s = lbm.Simulation("soa", lx, ly, 1, device=0, bc=bc, variant="fused2")
        s.init_rt_device(12345)
        s.step(0.8, 6)
        h = hashlib.sha1()
        if lx * ly <= 4096 * 2048:
            h.update(np.ascontiguousarray(s.dump()).tobytes())
        else:
            h.update(np.ascontiguousarray(s.moments()).tobytes())
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            s.step(0.8, n)
            best = min(best, time.perf_counter() - t0)
        s.close()
        res[var] = (best, h.hexdigest()[:12])
        print(f"{lx}x{ly} {bc:8s} form:sched {var}: {best / n * 1e3:.3f} ms/step = {lx * ly * n / best / 1e6:.0f} MLUPS "
              f"({lx * ly * 296 * n / best / 1e9:.0f} GB/s algorithmic) state {res[var][1]}", flush=True)
    first = next(iter(res.values()))
    print(f"  speed-up over the first: {' '.join(f'{k} {first[0] / v[0]:.3f}' for k, v in res.items())}  bitwise "
          f"{'same' if len({v[1] for v in res.values()}) == 1 else 'DIFFERENT'}", flush=True)
