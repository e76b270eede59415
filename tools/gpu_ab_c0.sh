# A/B on config 0 (256 x 1024, wall, 100-step calls) for caosoa32 and soa
V=${VARIANTS:-"new prev"}
for i in 1 2 3; do
  for v in $V; do
    timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so caosoa 32 fused 100 256 1024 2>&1 | tail -1 | sed 's/^/c0-caosoa32 /'
    timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so soa 1 fused 100 256 1024 2>&1 | tail -1 | sed 's/^/c0-soa /'
  done
done
