#!/bin/bash
# Builds an experimental variant of librsot_b200.so (extra -D flags) next to
# the default one: tools/build_variant.sh NAME -DFLAG ...  (development aid)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
C=paper_2507_23602_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -Iinclude "$@" -o paper_2507_23602_b200/lib/var_$name.so \
  $C/dense.cu $C/truncated.cu $C/refine.cu $C/geodesic.cu $C/capi.cu -ldl
