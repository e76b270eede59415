# ncu --set full of one FUSED2 bench sweep (k_step2_split) for the interior form $FORM (schedule $SCHED)
FORM=${FORM:-3}; SCHED=${SCHED:-1}; TAG=${TAG:-f${FORM}s${SCHED}}
mkdir -p gpurun_out/r02b
export D2Q37_STEP2_FORM=$FORM D2Q37_STEP2_SCHED=$SCHED
python tools/fused2_prof.py 4096 16384 > gpurun_out/r02b/p_$TAG.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:${KERNEL:-k_step2_split} -c 1 -o gpurun_out/r02b/prof_$TAG \
      python tools/fused2_prof.py 4096 16384 > gpurun_out/r02b/ncu_$TAG.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/r02b/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/r02b/prof_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/r02b/prof_$TAG.ncu-rep --page details --csv > gpurun_out/r02b/prof_${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/r02b/prof_$TAG.ncu-rep --page source --csv > gpurun_out/r02b/prof_${TAG}_source.csv 2>/dev/null
