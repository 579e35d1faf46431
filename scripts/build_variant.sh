#!/bin/bash
# Build an A/B variant of libks with extra nvcc defines: scripts/build_variant.sh NAME -DKS_PCG_THREADS=384 ...
# Output: paper_2404_19249_b200/libks_NAME.so (select with KS_LIB=...).
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude "$@" \
  -shared -cudart static -o paper_2404_19249_b200/libks_$NAME.so paper_2404_19249_b200/csrc/*.cu
