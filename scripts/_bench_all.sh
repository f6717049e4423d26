mkdir -p gpurun_out
TAG=${1:-r01h}
for c in c3 c3ir c3rw c1 c2 c4 c5_256 c5_4096 c5_65536; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err; echo "reference rc=$?"
