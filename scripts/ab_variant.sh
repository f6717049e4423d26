#!/bin/bash
# Build the working tree's libtaco with extra nvcc flags into
# build/ab/libtaco_<tag>.so (A/B of compile-time variants):
#   ab_variant.sh <tag> "-DTACO_SOMETHING=1 ..."
# then time it with TACO_LIB_PATH=build/ab/libtaco_<tag>.so.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build/ab"
(cd "$ROOT" && TACO_BUILD_OUT="$ROOT/build/ab/libtaco_$1.so" TACO_NVCC_EXTRA="${2:-}" \
   python -c "from paper_2404_04895_b200 import build; build.build_library(force=True)" > /dev/null)
echo "built $ROOT/build/ab/libtaco_$1.so"
