timeout 900 python -m paper_1804_01918_b200.bench_matrix --lx 1024 --ly 8192 --vl 8,32 --iterations 20 --warmup 3 \
    --energy -o gpurun_out/bench_matrix.csv 2> gpurun_out/bench_matrix.err; echo matrix rc=$?; cat gpurun_out/bench_matrix.err
timeout 300 python -m pytest tests/test_bench_matrix.py -q -m gpu 2>&1 | tail -2
