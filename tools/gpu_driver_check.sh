# what the driver runs at round end: smoke, the reference arm, the default bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_arm.log 2> gpurun_out/ref_arm.err; echo ref rc=$?; tail -1 gpurun_out/ref_arm.log
start=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench rc=$? elapsed=$(( $(date +%s) - start ))s
