#!/bin/bash
# Build an experimental variant of the library: tools/build_variant.sh NAME FILE.cu "-DMACRO=V ..."
# (FILE.cu recompiled with the extra defines, linked with the other objects
# of the regular build) -> paper_1707_07803_b200/lib/variants/libmpo_b200_NAME.so;
# select it at run time with MPO_B200_LIB=<that path>.
set -e
cd "$(dirname "$0")/.."
make -s
name=$1; src=$2; defs=$3
base=$(basename "$src" .cu)
mkdir -p build/variants/$name paper_1707_07803_b200/lib/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -Ipaper_1707_07803_b200/csrc \
  $defs -c paper_1707_07803_b200/csrc/$base.cu -o build/variants/$name/$base.o
objs=$(ls build/*.o | grep -v "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o paper_1707_07803_b200/lib/variants/libmpo_b200_$name.so $objs build/variants/$name/$base.o
echo paper_1707_07803_b200/lib/variants/libmpo_b200_$name.so
