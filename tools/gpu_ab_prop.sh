# A/B of the propagate verb on BASELINE config 1 (1024 x 8192), 200 calls, per layout
V=${VARIANTS:-"new prev"}
for i in 1 2 3; do
  for v in $V; do
    for lay in "caosoa 32" "soa 1"; do
      timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so $lay propagate 200 1024 8192 2>&1 | tail -1 | sed "s/^/c1-${lay% *} /"
    done
  done
done
