#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU): plain run, then the ncu launch
# list and full captures of the dominant kernels.  Outputs in gpurun_out/.
set -u
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_sorted -s 3 -c 1 \
    -o gpurun_out/prof_construct_sorted_$TAG $CMD > gpurun_out/ncu_sorted_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_row_update -s 6 -c 1 \
    -o gpurun_out/prof_row_update_$TAG $CMD > gpurun_out/ncu_row_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_construct_dense -c 1 \
    -o gpurun_out/prof_construct_dense_$TAG $CMD > gpurun_out/ncu_dense_$TAG.log 2>&1
RWCMD="python bench.py --config c3rw --steps 1 --warmup 3 --no-cpu-baseline"
$RWCMD > gpurun_out/plain_rw_$TAG.log 2>&1 || { echo "plain RW run failed"; tail -20 gpurun_out/plain_rw_$TAG.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_construct_rw -s 3 -c 1 \
    -o gpurun_out/prof_construct_rw_$TAG $RWCMD > gpurun_out/ncu_rw_$TAG.log 2>&1
ls -la gpurun_out/
