# ncu --set full of one steady-state fused step kernel for each A/B library.
V=${VARIANTS:-"new prev"}
for v in $V; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collide -s 30 -c 1 \
      -f -o gpurun_out/ab_$v python tools/ab_step.py tools/ab/libd2q37_b200_$v.so caosoa 32 fused 5 \
      > gpurun_out/ab_ncu_$v.log 2>&1; echo ncu $v rc=$?
done
