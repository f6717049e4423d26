#!/bin/bash
# Alternate the HEAD build (build/ab/libtaco_head.so) and the working-tree
# build: ab_time.sh <n> <m> <reps> [variant]
N=${1:-2392}; M=${2:-4096}; R=${3:-4}; V=${4:-sorted}
for r in $(seq 1 $R); do
  echo -n "head "; TACO_LIB_PATH=build/ab/libtaco_head.so timeout 120 python scripts/bench_construct.py --n $N --m $M --iters 3 --reps 5 --variant $V | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])"
  echo -n "work "; timeout 120 python scripts/bench_construct.py --n $N --m $M --iters 3 --reps 5 --variant $V | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])"
done
