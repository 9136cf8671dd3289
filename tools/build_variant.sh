#!/bin/bash
# usage: bash tools/build_variant.sh NAME [-DMACRO=V ...] -- build libfastspline_NAME.so (A/B tooling)
cd "$(dirname "$0")/.."
N=$1; shift
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -Iinclude -ldl "$@" \
  -o paper_2001_09253_b200/csrc/libfastspline_$N.so paper_2001_09253_b200/csrc/spline_abi.cu
