set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench2.log 2> gpurun_out/bench2.err; echo bench rc=$?; tail -2 gpurun_out/bench2.err
python profiles/profile_cmd.py --case step --steps 4 > gpurun_out/plain_step.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python profiles/profile_cmd.py --case step --steps 4 > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
python profiles/profile_cmd.py --case step --steps 3 > gpurun_out/plain_step3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_collide -s 1 -c 1 -o gpurun_out/prof_fused python profiles/profile_cmd.py --case step --steps 3 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
python profiles/profile_cmd.py --case collide --steps 3 > gpurun_out/plain_coll.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_collide -s 1 -c 1 -o gpurun_out/prof_collide python profiles/profile_cmd.py --case collide --steps 3 > gpurun_out/ncu_full2.log 2>&1; echo ncu3 rc=$?
python profiles/profile_cmd.py --case propagate --steps 3 > gpurun_out/plain_prop.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1 -c 1 -o gpurun_out/prof_propagate python profiles/profile_cmd.py --case propagate --steps 3 > gpurun_out/ncu_full3.log 2>&1; echo ncu4 rc=$?
tail -3 gpurun_out/ncu_full.log
