#!/bin/bash
# Build the committed HEAD's libtaco into build/ab/libtaco_head.so (A/B timing
# against the working tree's build: TACO_LIB_PATH selects the library).
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" worktree add -q --detach "$TMP" HEAD
(cd "$TMP" && python -m paper_2404_04895_b200.build > /dev/null)
mkdir -p "$ROOT/build/ab"
cp "$TMP/paper_2404_04895_b200/lib/libtaco.so" "$ROOT/build/ab/libtaco_head.so"
git -C "$ROOT" worktree remove --force "$TMP"
echo "built $ROOT/build/ab/libtaco_head.so"
