timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "nccl or slab or group" > gpurun_out/pytest_slab.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_slab.log
bash tools/gpu_slab_only.sh
