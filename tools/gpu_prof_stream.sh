# evidence for the streamed run: ncu launch list of one 20-step run (4096 x 16384 walls) and ncu --set full of
# one 37-band chunk sweep (the lockstep plan's even split: 4 CTAs per band)
mkdir -p gpurun_out/r02s
python tools/stream_run_prof.py 16384 20 > gpurun_out/r02s/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02s/launches_stream_run.csv \
      python tools/stream_run_prof.py 16384 20 > gpurun_out/r02s/ncu_launches.log 2>&1; echo launches rc=$?
# launch 60 of k_step2_pair in that run is a sweep of the first 37-band chunk
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step2_pair -s 60 -c 1 -o gpurun_out/r02s/prof_chunk_sweep \
      python tools/stream_run_prof.py 16384 20 > gpurun_out/r02s/ncu_chunk.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/r02s/prof_chunk_sweep.ncu-rep --page raw --csv > gpurun_out/r02s/prof_chunk_sweep_raw.csv 2>/dev/null
ncu -i gpurun_out/r02s/prof_chunk_sweep.ncu-rep --page details --csv > gpurun_out/r02s/prof_chunk_sweep_details.csv 2>/dev/null
ls gpurun_out/r02s
