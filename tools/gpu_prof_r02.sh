# round-2 evidence: bench launch list, ncu --set full of the bench sweep (k_step2_split), of the overlapped
# slab sweep (k_step2_slab) and of the halo kernels (k_pack6 serial schedule / k_unpack6)
mkdir -p gpurun_out/r02
ARGS="--steps 4 --warmup 4 --no-e2e --no-extras --no-cpu --no-other-scaling"
python bench.py $ARGS > gpurun_out/r02/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_bench.csv \
      python bench.py $ARGS > gpurun_out/r02/ncu_bench.log 2>&1; echo launches rc=$?
python tools/fused2_prof.py 4096 16384 > gpurun_out/r02/p1.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_step2_split -c 1 -o gpurun_out/r02/prof_step2_split \
      python tools/fused2_prof.py 4096 16384 > gpurun_out/r02/ncu_step2.log 2>&1; echo ncu1 rc=$?
python tools/fused2_slab_prof.py 4096 > gpurun_out/r02/p2.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_step2_slab|k_unpack6|k_pack6" -c 4 -o gpurun_out/r02/prof_slab \
      python tools/fused2_slab_prof.py 4096 > gpurun_out/r02/ncu_slab.log 2>&1; echo ncu2 rc=$?
for f in gpurun_out/r02/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
done
ls -la gpurun_out/r02
