# A/B(/C) the single-domain step: tools/ab/libd2q37_b200_<v>.so, alternated to cancel drift.
# usage: VARIANTS="new prev" bash tools/gpu_ab.sh [layout vl variant]
V=${VARIANTS:-"new prev"}
for i in 1 2 3; do
  for v in $V; do
    timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so "$@" 2>&1 | tail -1
  done
done
