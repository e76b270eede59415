# round-2 evidence for the final pair-form sweep: bench line, bench launch list, ncu --set full of one bench sweep
# (k_step2_pair, 4096 x 16384 walls) and of the overlapped slab sweep (k_step2_pair_slab, 1-rank NCCL ring)
mkdir -p gpurun_out/r02g
python bench.py > gpurun_out/r02g/bench_default.json 2> gpurun_out/r02g/bench_default.err; echo bench rc=$?
ARGS="--steps 4 --warmup 4 --no-e2e --no-extras --no-cpu --no-other-scaling"
python bench.py $ARGS > gpurun_out/r02g/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02g/launches_bench.csv \
      python bench.py $ARGS > gpurun_out/r02g/ncu_bench.log 2>&1; echo launches rc=$?
python tools/fused2_prof.py 4096 16384 > gpurun_out/r02g/p1.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step2_pair -c 1 -o gpurun_out/r02g/prof_step2_pair \
      python tools/fused2_prof.py 4096 16384 > gpurun_out/r02g/ncu_pair.log 2>&1; echo ncu1 rc=$?
python tools/fused2_slab_prof.py 4096 > gpurun_out/r02g/p2.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step2_pair_slab -c 1 -o gpurun_out/r02g/prof_pair_slab \
      python tools/fused2_slab_prof.py 4096 > gpurun_out/r02g/ncu_slab.log 2>&1; echo ncu2 rc=$?
for f in gpurun_out/r02g/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
done
ls gpurun_out/r02g
# source-level stall samples of the sweep kernel (SASS view) and the reference arm
ncu -i gpurun_out/r02g/prof_step2_pair.ncu-rep --page source --csv --print-source sass > gpurun_out/r02g/prof_step2_pair_source_sass.csv 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02g/bench_reference.json 2> gpurun_out/r02g/bench_reference.err; echo ref rc=$?
