mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_banded.py -q -x > gpurun_out/g4_pytest.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/g4_pytest.log
BC=wall timeout 300 python tools/fused2_banded_time.py > gpurun_out/g4_time.log 2>&1; echo time rc=$?; cat gpurun_out/g4_time.log
