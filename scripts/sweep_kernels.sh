#!/bin/bash
# Construction time of every sorted-kernel instantiation at the given sizes:
#   sweep_kernels.sh "<n>x<m> ..."
for cfg in $1; do
  N=${cfg%x*}; M=${cfg#*x}
  for k in ${KERNELS:-warp g16e2 g8e2 g8e4 g4e2 g4e4}; do
    ms=$(TACO_SORTED_KERNEL=$k timeout 300 python scripts/bench_construct.py --n $N --m $M --iters 3 --reps 5 | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])")
    echo "$cfg $k $ms"
  done
done
