#!/bin/bash
# Build a perf-experiment variant of the library: tools/build_variant.sh NAME -DFLAG=V ...
# -> paper_2605_19926_b200/variant_NAME.so (select with TILECAST_B200_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  --fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC -shared "$@" \
  "$ROOT/paper_2605_19926_b200/csrc/tilecast_b200.cu" -o "$ROOT/paper_2605_19926_b200/variant_$name.so"
