# full GPU suite + the device bench matrix CSV (reference schema v1, NVML energy)
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python -m paper_1804_01918_b200.bench_matrix --lx 1024 --ly 8192 --vl 8,32 --iterations 20 --warmup 3 \
    --energy -o gpurun_out/bench_matrix.csv 2> gpurun_out/bench_matrix.err; echo matrix rc=$?; cat gpurun_out/bench_matrix.err
