#!/bin/bash
# Builds the sweep-kernel cycle-profile variant of the library into tools/prof_lib/ (use with
# RNMF_GPU_LIB=tools/prof_lib/librnmf_gpu.so RNMF_PROF=1).  Development aid only.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/paper_1711_02037_b200" "$ROOT/tools/prof_lib"
cp -r "$ROOT/paper_1711_02037_b200/csrc" "$TMP/paper_1711_02037_b200/"
cp -r "$ROOT/include" "$TMP/"
rm -rf "$TMP/paper_1711_02037_b200/csrc/build"
make -s -C "$TMP/paper_1711_02037_b200/csrc" -j8 EXTRA=-DRNMF_SWEEP_PROF=1 OUT="$ROOT/tools/prof_lib/librnmf_gpu.so"
rm -rf "$TMP"
