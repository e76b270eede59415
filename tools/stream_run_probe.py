"""Sweeps-only timing (D2Q37_STREAM_PROBE=1) of the streamed run for several chunk heights.
usage: python tools/stream_run_probe.py [ROWS:FIRST:LAST ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1804_01918_b200 as lbm  # noqa: E402

lx, ly, n = 4096, 16384, int(os.environ.get("PROBE_STEPS", "200"))
combos = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(4080, 480, 240)]
s = lbm.Simulation("soa", lx, ly, device=0, bc="wall", variant="fused2")
s.init_rt_device(2018)
canon = np.empty((37, lx, ly))
assert int(torch.cuda.cudart().cudaHostRegister(canon.ctypes.data, canon.nbytes, 0)) == 0
s.dump(out=canon)
for probe in (1, 3, 4, 0):
    os.environ["D2Q37_STREAM_PROBE"] = str(probe)
    for rows, first, last in combos:
        os.environ["D2Q37_STREAM_ROWS"] = str(rows)
        os.environ["D2Q37_STREAM_FIRST"] = str(first)
        os.environ["D2Q37_STREAM_LAST"] = str(last)
        best = 1e30
        for _ in range(3):
            if probe:
                s.init_rt_device(2018)
            t0 = time.perf_counter()
            s.run(canon, 0.8, n, out=canon)
            best = min(best, time.perf_counter() - t0)
        print(f"probe {probe} rows {rows} first {first} last {last}: {best:.4f} s {lx * ly * n / best / 1e6:.0f} MLUPS",
              flush=True)
