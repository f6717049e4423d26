for m in 4096 2048 8192; do
 for T in 0 4 8; do
  for L in 0 1; do
   if [ $T = 0 ] && [ $L = 1 ]; then continue; fi
   TACO_SORTED_T=$T TACO_LAZY=$L timeout 120 python scripts/bench_construct.py --n 2392 --m $m --iters 5 --reps 5 | sed "s/^/T=$T L=$L /"
  done
 done
done
