for i in 1 2; do
  for v in base probe3 probe6 probe7; do
   AB_IGNORE_ERRORS=1 timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so banded 1 fused2 40 2>&1 | tail -1
  done
done
