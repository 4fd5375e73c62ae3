#!/bin/bash
# Build an A/B variant of the library with extra nvcc defines into build/variants/<name>/
# usage: tools/build_variant.sh NAME "-DKS_ST_NS=6 -DKS_ST_MINB=3" [SRCDIR]   (select with KS_LIB=... at run time)
# SRCDIR (default paper_2604_25422_b200/csrc): e.g. a checkout of an older revision's csrc for an A/B
set -e
NAME=$1; DEFS=$2; SRC=${3:-paper_2604_25422_b200/csrc}
D=build/variants/$NAME
mkdir -p $D/obj
for f in $SRC/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Iinclude \
    -I$SRC --expt-relaxed-constexpr $DEFS -c $f -o $D/obj/$b.o &
done
g++ -O2 -std=c++20 -fPIC -Iinclude -I/usr/local/cuda/include -c $SRC/conv_core.cpp -o $D/obj/conv_core.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libks_dwconv1d.so $D/obj/*.o -lnccl -Xlinker -soname=libks_dwconv1d.so
rm -rf $D/obj
echo built $D/libks_dwconv1d.so
