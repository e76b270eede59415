import sys, json
sys.path.insert(0, ".")
import bench, paper_1804_01918_b200 as lbm
print(json.dumps(bench.bench_fused2_group_emulation(lbm, 8, 4, 20)))
