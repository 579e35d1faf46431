#!/bin/bash
# Build an A/B variant of libks with extra nvcc defines: scripts/build_variant.sh NAME -DKS_PCG_THREADS=384 ...
# Output: paper_2404_19249_b200/libks_NAME.so (select with KS_LIB=...). Same compile flags and link line
# (cuSOLVER, cuBLAS, toolkit rpath) as the default build (paper_2404_19249_b200/_build.py).
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
python -c "import sys; from paper_2404_19249_b200 import _build; \
_build.build(force=True, verbose=True, defines=sys.argv[2:], out='paper_2404_19249_b200/libks_'+sys.argv[1]+'.so')" "$NAME" "$@"
