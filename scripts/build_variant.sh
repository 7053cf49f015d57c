#!/bin/bash
# Build libtomo from a git revision (default HEAD) into paper_2104_12282_b200/lib/<name>.so
# for A/B timing: TOMO_LIB_PATH=$PWD/paper_2104_12282_b200/lib/<name>.so python bench.py ...
set -e
REV=${1:-HEAD}; NAME=${2:-libtomo_ref}; shift 2 || true
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2104_12282_b200/csrc include | tar -x -C "$TMP"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  -Xcompiler -fPIC -shared -cudart static -I "$TMP/include" "$@" \
  $(ls "$TMP"/paper_2104_12282_b200/csrc/*.cu) \
  -o "$ROOT/paper_2104_12282_b200/lib/$NAME.so"
rm -rf "$TMP"
echo "$ROOT/paper_2104_12282_b200/lib/$NAME.so"
