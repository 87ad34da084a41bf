#!/bin/bash
# Build a compile-flag variant of the library into gpuvar/<name>.so (CPU side):
#   tools/variant.sh <name> "<nvcc flags>"
# and compare variants on the GPU box with tools/variant_bench.sh.
set -e
name=$1; flags=$2
mkdir -p gpuvar
PXST_BUILD_DIR=build/var_$name PXST_LIB_OUT=$PWD/gpuvar/$name.so PXST_NVCC_EXTRA="$flags" \
  python -c "import sys; sys.path.insert(0, '.'); from paper_2003_12726_b200 import build_native as b; b.build()"
ls -la gpuvar/$name.so
