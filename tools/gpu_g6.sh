mkdir -p gpurun_out
timeout 120 python tools/fused2_banded_prof.py 4096 4096 > gpurun_out/g6_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_band_sweep -c 1 -o gpurun_out/prof_band2 \
    python tools/fused2_banded_prof.py 4096 4096 > gpurun_out/g6_ncu.log 2>&1; echo ncu rc=$?
