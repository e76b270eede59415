mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "nccl or slab or fused2" > gpurun_out/g9_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/g9_pytest.log
for v in 1 0; do D2Q37_STEP2_OVERLAP=$v timeout 600 python tools/fused2_slab_overlap.py 4096 16384 2>&1 | grep -v NCCL | sed "s/^/overlap=$v /"; done
for m in 0 2; do D2Q37_STEP2_HALO_SMS=$m timeout 600 python tools/fused2_slab_overlap.py 4096 2>&1 | grep -v NCCL | sed "s/^/halo_sms=$m /"; done
