#!/bin/bash
# Build a tuning variant of libLBX: scripts/build_variant.sh NAME -DFLAG=V ...
name=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off,-O3,-fopenmp -lgomp -shared -Iinclude "$@" \
  paper_2104_11385_b200/csrc/*.cu paper_2104_11385_b200/csrc/*.cpp \
  -o paper_2104_11385_b200/libLBX.$name.so
