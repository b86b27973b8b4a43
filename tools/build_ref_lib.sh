#!/bin/bash
# Experiment helper: build libmpsf.so from a git revision (default HEAD) into build/var/libmpsf_<name>.so,
# for A/B runs against the working tree (tools/variants.py run ... <name> prod).
set -e
REV=${1:-HEAD}; NAME=${2:-base}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2605_26461_b200/csrc include | tar -x -C "$TMP"
mkdir -p "$ROOT/build/var"
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 -I "$TMP/include" \
  -shared -o "$ROOT/build/var/libmpsf_$NAME.so" "$TMP"/paper_2605_26461_b200/csrc/*.cu "$TMP"/paper_2605_26461_b200/csrc/*.cpp
rm -rf "$TMP"
echo "built build/var/libmpsf_$NAME.so from $REV"
