"""A 1-rank NCCL FUSED2 ring on 4096 x 4096 (the 8-GPU strong slab), for ncu (-k regex:k_step2_slab|k_unpack6|k_pack6)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: F401,E402  (torch's libnccl.so.2)

import paper_1804_01918_b200 as lbm  # noqa: E402

ly = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = lbm.Simulation.slab("soa", 4096, ly, 1, device=0, rank=0, nranks=1, nccl_id=lbm.nccl_unique_id(),
                        bc="periodic", variant="fused2")
s.init_rt_device(12345)
s.step(0.8, 6)
s.sync()
