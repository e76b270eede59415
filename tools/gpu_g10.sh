mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ymajor or nccl_self_ring" > gpurun_out/g10.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/g10.log
