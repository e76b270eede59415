mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_banded.py -q -x > gpurun_out/g5_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/g5_pytest.log
BC=wall timeout 300 python tools/fused2_banded_time.py > gpurun_out/g5_time.log 2>&1; echo time rc=$?; cat gpurun_out/g5_time.log
timeout 120 python tools/fused2_banded_prof.py 4096 16384 > gpurun_out/g5_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_band_sweep -c 1 -o gpurun_out/prof_band \
    python tools/fused2_banded_prof.py 4096 16384 > gpurun_out/g5_ncu.log 2>&1; echo ncu rc=$?
