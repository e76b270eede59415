"""Timeline of the overlapped FUSED2 slab sweep through a real 1-rank NCCL ring (CUDA events on the lattice
and comm streams, d2q37_slab_timeline): when the 6-row halo exchange starts, when NCCL and the unpack end,
and when the sweep ends -- the evidence that the exchange runs under the interior.
usage: python tools/slab_timeline.py [lx ly ...]"""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402,F401  (torch's libnccl.so.2)
import paper_1804_01918_b200 as lbm  # noqa: E402

a = [int(v) for v in sys.argv[1:]] or [4096, 16384, 4096, 4096]
for lx, ly in zip(a[0::2], a[1::2]):
    s = lbm.Simulation.slab("soa", lx, ly, 1, rank=0, nranks=1, nccl_id=lbm.nccl_unique_id(), bc="periodic",
                            variant="fused2")
    s.init_rt_device(12345)
    s.step(0.8, 4)
    s.set_profiling(True)
    rows = []
    for _ in range(5):
        s.step(0.8, 2)
        rows.append(s.slab_timeline())
    s.set_profiling(False)
    s.close()
    best = min(rows, key=lambda r: r["sweep_done"])
    print(json.dumps({"slab": f"{lx}x{ly}", "transport": "nccl (1-rank ring)", "ms_after_sweep_launch": best,
                      "exchange_hidden": best["unpack_done"] <= best["sweep_done"],
                      "exchange_start_frac_of_sweep": best["exchange_start"] / best["sweep_done"]}), flush=True)
