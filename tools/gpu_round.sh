# one gpurun round: GPU parity tests, then the bench (plain, no profiler)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 50 --warmup 5 --no-e2e --no-cpu} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?; tail -3 gpurun_out/bench.err
