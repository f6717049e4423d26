#!/bin/bash
# Alternate construction timings of several libtaco builds (A/B):
#   ab_libs.sh "<lib1> <lib2> ..." "<n>x<m> ..." [reps] [variant]
# A lib path "work" means the working tree's paper_2404_04895_b200/lib/libtaco.so.
LIBS=$1; CFGS=$2; R=${3:-3}; V=${4:-sorted}
for cfg in $CFGS; do
  N=${cfg%x*}; M=${cfg#*x}
  for r in $(seq 1 $R); do
    for lib in $LIBS; do
      if [ "$lib" = work ]; then unset TACO_LIB_PATH; else export TACO_LIB_PATH=$lib; fi
      ms=$(timeout 300 python scripts/bench_construct.py --n $N --m $M --iters 3 --reps 5 --variant $V | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms'])")
      echo "$cfg $lib $ms"
    done
  done
done
unset TACO_LIB_PATH
