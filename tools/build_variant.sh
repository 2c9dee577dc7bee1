#!/bin/bash
# Build an alternate library with compile-time overrides: build_variant.sh NAME "-DFOO=1 -DBAR=2"
# Only recompiles the given sources (default: all); ptxas report in $OUT/ptxas.txt.
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
OUT=build/var_$NAME; mkdir -p $OUT
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -I include $DEFS"
for f in paper_2204_02064_b200/csrc/*.cu; do nvcc $FL -c $f -o $OUT/$(basename $f).o 2> $OUT/$(basename $f).ptxas & done; wait
cat $OUT/*.ptxas > $OUT/ptxas.txt
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT/libperks_stencil.so $OUT/*.o -lcudart
echo $OUT/libperks_stencil.so
