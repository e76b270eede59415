"""FUSED2 y-slab schedule on one GPU: 1-rank NCCL ring (6-row halos through ncclSend/Recv to self)
vs the single domain, at the 8-GPU strong slab (4096 x 4096) and the weak slab (4096 x 16384)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402,F401  (torch's libnccl.so.2)
import paper_1804_01918_b200 as lbm  # noqa: E402

for ly in (4096, 16384):
    out = {}
    for name in ("single", "nccl_ring"):
        if name == "single":
            s = lbm.Simulation("soa", 4096, ly, 1, device=0, bc="periodic", variant="fused2")
        else:
            s = lbm.Simulation.slab("soa", 4096, ly, 1, rank=0, nranks=1, nccl_id=lbm.nccl_unique_id(),
                                    bc="periodic", variant="fused2")
        s.init_rt_device(12345)
        s.step(0.8, 4)
        n = 40
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            s.step(0.8, n)
            best = min(best, time.perf_counter() - t0)
        out[name] = best / n * 1e3
        if name != "single":
            out["exposed_halo_ms_per_sweep"] = s.exposed_halo_ms()
        s.close()
    print(f"4096x{ly}: single {out['single']:.3f} ms/step, NCCL ring {out['nccl_ring']:.3f} ms/step "
          f"(+{(out['nccl_ring'] / out['single'] - 1) * 100:.2f} %), exposed halo {out['exposed_halo_ms_per_sweep']:.3f} ms/sweep",
          flush=True)
