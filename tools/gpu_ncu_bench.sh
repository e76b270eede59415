# ncu launch list of the bench command itself (plain run first, same args)
ARGS="--steps 3 --warmup 3 --no-e2e --no-extras --no-cpu"
python bench.py $ARGS > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
      python bench.py $ARGS > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/bench_plain.log
