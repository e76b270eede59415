# GPU tests + default bench + ncu evidence for the CAoSoA32 fused step kernel (bench default)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?; tail -3 gpurun_out/bench.err
python profiles/profile_cmd.py --case caosoa --steps 4 > gpurun_out/plain_caosoa.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_caosoa.csv python profiles/profile_cmd.py --case caosoa --steps 4 > gpurun_out/ncu_launch_caosoa.log 2>&1; echo ncu1 rc=$?
python profiles/profile_cmd.py --case caosoa --steps 3 > gpurun_out/plain_caosoa3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_collide -s 1 -c 1 -o gpurun_out/prof_fused_caosoa python profiles/profile_cmd.py --case caosoa --steps 3 > gpurun_out/ncu_full_caosoa.log 2>&1; echo ncu2 rc=$?
