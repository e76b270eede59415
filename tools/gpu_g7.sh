for i in 1 2; do
 for lay in soa banded; do
  for v in base split; do
   timeout 300 python tools/ab_step.py tools/ab/libd2q37_b200_$v.so $lay 1 fused2 40 2>&1 | tail -1 | sed "s/^/$lay /"
  done
 done
done
