"""One streamed run (Simulation.run) of NSTEPS steps on 4096 x LY walls with a pinned host canonical, for
ncu launch lists / captures.  usage: python tools/stream_run_prof.py [LY] [NSTEPS]"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1804_01918_b200 as lbm  # noqa: E402

ly = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
s = lbm.Simulation("soa", 4096, ly, device=0, bc=os.environ.get("BC", "wall"), variant="fused2")
s.init_rt_device(2018)
canon = np.empty((37, 4096, ly))
assert int(torch.cuda.cudart().cudaHostRegister(canon.ctypes.data, canon.nbytes, 0)) == 0
s.dump(out=canon)
s.run(canon, 0.8, n, out=canon)
print(s.last_run_mode)
