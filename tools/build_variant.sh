#!/bin/bash
# usage: tools/build_variant.sh <name> [nvcc -D flags...]  -> build_ab/<name>.so (A/B experiments)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/build_ab"
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Xptxas -warn-spills "$@" "$ROOT/paper_2205_15401_b200/csrc/gvr_cuda.cu" -o "$ROOT/build_ab/$name.so" 2>&1 | grep -v "^$" | grep -i "spill\|error" | grep -v " 0 bytes spill stores" | grep "Li20E\|error" || true
