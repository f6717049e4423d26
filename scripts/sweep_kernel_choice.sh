for m in 6144 8192 12288; do
  for k in warp g8e2 g4e4; do
    echo -n "$m $k "; TACO_SORTED_KERNEL=$k timeout 120 python scripts/bench_construct.py --n 2392 --m $m --iters 3 --reps 3 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])"
  done
done
for k in warp g8e2 g4e4; do echo -n "5000x65536 $k "; TACO_SORTED_KERNEL=$k timeout 300 python scripts/bench_construct.py --n 5000 --m 65536 --iters 2 --reps 2 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])"; done
