for i in 1 2; do
 for f in 0 2; do
  for v in o122 o120; do
   D2Q37_STEP2_FORM=$f timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so soa 1 fused2 40 2>&1 | tail -1 | sed "s/^/form $f /"
  done
 done
done
