# lockstep schedule evidence: membench pattern ceilings (lock 0/1, 1-4 stages) and ncu --set full of the lockstep sweep
mkdir -p gpurun_out/r02b
(cd tools/experiments/tb2 && timeout 300 ./membench 4096 16384) > gpurun_out/r02b/membench_lock.log 2>&1; echo membench rc=$?
python tools/fused2_prof.py 4096 16384 > gpurun_out/r02b/p1.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step2_split -c 1 -o gpurun_out/r02b/prof_step2_lock \
      python tools/fused2_prof.py 4096 16384 > gpurun_out/r02b/ncu_lock.log 2>&1; echo ncu rc=$?
for f in gpurun_out/r02b/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
done
