timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "full_size" --durations=5 > gpurun_out/pytest_full.log 2>&1; echo rc=$?; tail -12 gpurun_out/pytest_full.log
