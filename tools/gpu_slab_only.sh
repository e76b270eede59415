# quick: only the slab-schedule sub-bench
timeout 600 python - > gpurun_out/slab.log 2>&1 <<'PY'
import json, sys
sys.path.insert(0, ".")
import bench, paper_1804_01918_b200 as lbm
print(json.dumps(bench.bench_slab_schedule(lbm, "caosoa", 32, 4096, 3, 50), indent=1))
print(json.dumps(bench.bench_slab_schedule(lbm, "soa", 1, 4096, 3, 50), indent=1))
PY
echo rc=$?; cat gpurun_out/slab.log
