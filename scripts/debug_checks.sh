#!/bin/bash
# In place of compute-sanitizer (closed on this GPU pool): build libtaco with
# -DTACO_DEBUG_CHECKS (device traps on any out-of-range city / column index a
# kernel is about to use) and run the GPU suite and the kernel smoke against
# it.  A failed check prints "TACO_DCHECK failed: ..." and kills the context.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
scripts/ab_variant.sh debug "-DTACO_DEBUG_CHECKS" > /dev/null || exit 1
export TACO_LIB_PATH=$ROOT/build/ab/libtaco_debug.so
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python scripts/kernel_smoke.py 2>&1 | tail -2
