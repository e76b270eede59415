"""Times the streamed run (Simulation.run) against load + step + dump on 4096 x LY walls, pinned host
canonical, for a list of chunk heights.  usage: python tools/stream_run_time.py [LY] [NSTEPS] [ROWS:FIRST:LAST ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1804_01918_b200 as lbm  # noqa: E402

ly = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
combos = [tuple(int(v) for v in a.split(":")) for a in sys.argv[3:]] or [(4080, 480, 240)]
lx = 4096
bc = os.environ.get("BC", "wall")  # wall | periodic
s = lbm.Simulation("soa", lx, ly, device=0, bc=bc, variant="fused2")
s.init_rt_device(2018)
canon = np.empty((37, lx, ly))
assert int(torch.cuda.cudart().cudaHostRegister(canon.ctypes.data, canon.nbytes, 0)) == 0
s.dump(out=canon)


def timed(call, reps=2):
    best = 1e30
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        call()
        best = min(best, time.perf_counter() - t0)
    return best


def three():
    s.load(canon)
    s.step(0.8, n)
    s.dump(out=canon)


t = timed(three)
print(f"three verbs: {t:.4f} s  {lx * ly * n / t / 1e6:.0f} MLUPS", flush=True)
t = timed(lambda: s.step(0.8, n))
print(f"steps only:  {t:.4f} s  {lx * ly * n / t / 1e6:.0f} MLUPS", flush=True)
for rows, first, last in combos:
    os.environ["D2Q37_STREAM_ROWS"] = str(rows)
    os.environ["D2Q37_STREAM_FIRST"] = str(first)
    os.environ["D2Q37_STREAM_LAST"] = str(last)
    t = timed(lambda: s.run(canon, 0.8, n, out=canon))
    print(f"streamed ({s.last_run_mode}) rows {rows} first {first} last {last}: {t:.4f} s  "
          f"{lx * ly * n / t / 1e6:.0f} MLUPS", flush=True)
for probe, what in ((1, "sweeps only (no copies)"), (2, "copies only (no sweeps)")):
    os.environ["D2Q37_STREAM_PROBE"] = str(probe)
    t = timed(lambda: s.run(canon, 0.8, n, out=canon))
    print(f"probe {what}: {t:.4f} s", flush=True)
