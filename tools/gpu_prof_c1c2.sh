# ncu --set full of the propagate (config 1) and collide (config 2) kernels, SoA and CAoSoA32
for lay in "soa 1" "caosoa 32"; do
  set -- $lay
  for case in propagate collide; do
    python profiles/profile_cmd.py --case $case --layout $1 --vl $2 --steps 3 > gpurun_out/plain_${case}_$1.log 2>&1 && \
      ncu --set full --clock-control none --import-source on -k regex:k_ -s 2 -c 1 -f \
          -o gpurun_out/prof_${case}_$1 python profiles/profile_cmd.py --case $case --layout $1 --vl $2 --steps 3 \
          > gpurun_out/ncu_${case}_$1.log 2>&1; echo ncu $case $1 rc=$?
  done
done
# export on the box (the .ncu-rep files together exceed gpurun's 64 MiB merge limit)
for f in gpurun_out/prof_propagate_* gpurun_out/prof_collide_*; do
  case $f in *.ncu-rep)
    b=${f%.ncu-rep}
    ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
    ncu -i $f --page details --csv > ${b}_details.csv 2>/dev/null
    rm -f $f ;;
  esac
done
ls -la gpurun_out | head -30
