"""Streamed run against load + step + dump over lattice heights and step counts (default plan).
usage: [BC=wall|periodic] python tools/stream_run_shapes.py [LY:N ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1804_01918_b200 as lbm  # noqa: E402

lx = 4096
combos = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(16384, 200)]
for ly, n in combos:
    s = lbm.Simulation("soa", lx, ly, device=0, bc=os.environ.get("BC", "wall"), variant="fused2")
    s.init_rt_device(2018)
    canon = np.empty((37, lx, ly))
    assert int(torch.cuda.cudart().cudaHostRegister(canon.ctypes.data, canon.nbytes, 0)) == 0
    s.dump(out=canon)
    res = {}
    for name in ("streamed", "verbs"):
        best = 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            if name == "streamed":
                s.run(canon, 0.8, n, out=canon)
            else:
                s.load(canon)
                s.step(0.8, n)
                s.dump(out=canon)
            best = min(best, time.perf_counter() - t0)
        res[name] = best
    s.step(0.8, n)
    s.sync()
    t0 = time.perf_counter()
    s.step(0.8, n)
    s.sync()
    dev = time.perf_counter() - t0
    floor = max(dev, res["verbs"] - dev) if res["verbs"] > dev else dev  # the slower of the steps and the copies
    flag = "  <-- SLOW" if res["streamed"] > 1.25 * floor + 0.03 else ""
    print(f"ly {ly} n {n}: streamed {res['streamed']:.4f} s, three verbs {res['verbs']:.4f} s, steps alone {dev:.4f} s "
          f"(after the last call: {s.last_run_mode}){flag}", flush=True)
    torch.cuda.cudart().cudaHostUnregister(canon.ctypes.data)
    s.close()
    del canon
