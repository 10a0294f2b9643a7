#!/bin/bash
# Build one variant of the library with extra -D flags into build/<name>.so
# usage: bash tools/build_variant.sh <name> [srcdir] -DFOO=1 ...
NAME=$1; shift
SRC=${1:-paper_2105_00039_b200/csrc}; shift
mkdir -p build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O2 "$@" -shared -o build/$NAME.so $SRC/cellgrid_b200.cu
