#!/bin/bash
# Build an alternate library with compile-time overrides: build_variant.sh NAME "-DFOO=1 -DBAR=2" [src.cu ...]
# Recompiles only the given sources (default: all); the others are taken from the main build/.
# ptxas report in $OUT/ptxas.txt.
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2; shift 2
OUT=build/var_$NAME; mkdir -p $OUT
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -I include $DEFS"
SRCS=${@:-paper_2204_02064_b200/csrc/*.cu}
for f in paper_2204_02064_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  if [[ " $SRCS " == *" $f "* || " $SRCS " == *" $(basename $f) "* ]]; then
    nvcc $FL -c $f -o $OUT/$b.cu.o 2> $OUT/$b.ptxas &
  else
    cp build/$b.cu.o $OUT/$b.cu.o
  fi
done; wait
cat $OUT/*.ptxas > $OUT/ptxas.txt 2>/dev/null || true
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT/libperks_stencil.so $OUT/*.o -lcudart
echo $OUT/libperks_stencil.so
