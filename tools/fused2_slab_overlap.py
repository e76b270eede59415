"""FUSED2 y-slab schedule on one GPU: a 1-rank NCCL ring (overlapped halo pipeline) vs the single domain.
Usage: python tools/fused2_slab_overlap.py [ly ...]   (D2Q37_STEP2_OVERLAP=0: the serial schedule)"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1804_01918_b200 as lbm  # noqa: E402

for ly in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    for rep in range(2):
        r = bench.bench_slab_schedule_fused2(lbm, ly, 4, 40 if ly <= 4096 else 20)
        print(json.dumps({"ly": ly, "rep": rep, "overhead": r["schedule_overhead"],
                          "single_ms": r["single_domain"]["ms_per_step"],
                          "ring_ms": r["nccl_self_ring"]["ms_per_step"],
                          "exposed_halo_ms_per_step": r["nccl_self_ring"]["exposed_halo_ms_per_step"]}), flush=True)
