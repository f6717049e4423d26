timeout 900 python -m pytest tests -m gpu -q -k "dense or variant or parity" 2>&1 | tail -2
run() { timeout 300 python scripts/bench_construct.py --variant dense --n $1 --m $2 --iters 3 --reps 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms'], d['tour_checksum'])"; }
for cfg in "2392 4096" "1000 1024"; do set -- $cfg
  echo -n "$1 $2 head "; TACO_LIB_PATH=build/ab/libtaco_head.so run $1 $2; echo -n "$1 $2 work "; run $1 $2
done
