# FUSED2 bench check + ncu evidence of k_step2 at the bench size
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 4 --no-extras --no-cpu --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench rc=$?
ARGS="--steps 4 --warmup 4 --no-e2e --no-extras --no-cpu"
python bench.py $ARGS > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_step2.csv \
      python bench.py $ARGS > gpurun_out/ncu_bench.log 2>&1; echo launches rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_step2_split -c 1 -o gpurun_out/prof_step2_soa \
    python tools/fused2_prof.py 4096 16384 > gpurun_out/ncu_step2.log 2>&1; echo ncu rc=$?
