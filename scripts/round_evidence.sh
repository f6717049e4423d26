#!/bin/bash
# Round-end evidence in one gpurun call (outputs in gpurun_out/, copied to
# profiles/ by hand):  round_evidence.sh <tag>
#   bench lines of every config, the reference arm (C3 sampled, C1 as-is),
#   the scaling projections, and the ncu launch list + sorted-kernel captures
#   (C3, C4) + row-update capture (C3) of the same build.
TAG=${1:-r02p}
mkdir -p gpurun_out
for c in c3 c3ir c3rw c1 c2 c4 c5_256 c5_4096 c5_65536; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
echo "reference rc=$?"
timeout 900 python bench.py --impl reference --config c1 > gpurun_out/${TAG}_bench_reference_c1.json 2> gpurun_out/${TAG}_bench_reference_c1.err
echo "reference c1 rc=$?"
python scripts/project_scaling.py --n 2392 --m 4096 --out gpurun_out/${TAG}_projection_c3.json > /dev/null 2>&1; echo "proj c3 rc=$?"
python scripts/project_scaling.py --n 10000 --m 8192 --sel ir --out gpurun_out/${TAG}_projection_c4.json > /dev/null 2>&1; echo "proj c4 rc=$?"
scripts/profile_round.sh $TAG launches > /dev/null 2>&1; echo "launches rc=$?"
scripts/profile_round.sh $TAG sorted > /dev/null 2>&1; echo "sorted rc=$?"
CONFIG=c4 scripts/profile_round.sh ${TAG}c4 sorted > /dev/null 2>&1; echo "sorted c4 rc=$?"
scripts/profile_round.sh ${TAG}row row > /dev/null 2>&1; echo "row rc=$?"
