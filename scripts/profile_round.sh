#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU), one ncu pass per gpurun call:
#   profile_round.sh <tag> launches|sorted|row|dense|rw
# Each call first runs the same command without ncu (it must exit 0), then
# the one ncu pass: the launch list, or one --set full capture of a dominant
# kernel.  Outputs in gpurun_out/.
set -u
TAG=${1:-r01}
WHAT=${2:-launches}
CONFIG=${CONFIG:-c3}
CMD="python bench.py --config $CONFIG --steps 2 --warmup 1 --no-cpu-baseline"
RWCMD="python bench.py --config c3rw --steps 1 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
if [ "$WHAT" = rw ]; then RUN=$RWCMD; else RUN=$CMD; fi
$RUN > gpurun_out/plain_${WHAT}_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_${WHAT}_$TAG.log; exit 1; }
FULL="ncu --set full --clock-control none --import-source on"
case $WHAT in
  launches) ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
              --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1 ;;
  sorted) $FULL -k regex:k_construct_sorted -s 3 -c 1 -o gpurun_out/prof_construct_sorted_$TAG $CMD \
            > gpurun_out/ncu_sorted_$TAG.log 2>&1 ;;
  row) $FULL -k regex:k_row_update -s 6 -c 1 -o gpurun_out/prof_row_update_$TAG $CMD \
         > gpurun_out/ncu_row_$TAG.log 2>&1 ;;
  dense) $FULL -k regex:k_construct_dense -c 1 -o gpurun_out/prof_construct_dense_$TAG $CMD \
           > gpurun_out/ncu_dense_$TAG.log 2>&1 ;;
  rw) $FULL -k regex:k_construct_rw -s 3 -c 1 -o gpurun_out/prof_construct_rw_$TAG $RWCMD \
        > gpurun_out/ncu_rw_$TAG.log 2>&1 ;;
esac
echo "ncu rc=$?"
ls -la gpurun_out/ | grep $TAG
