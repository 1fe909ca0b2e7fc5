#!/bin/bash
# Build variants of the device library that differ in one source file's
# compile flags: tools/ab_build.sh FILE NAME:"-DFLAG=1" ... -> paper_1903_06631_b200/ab/lib_NAME.so
set -e
cd "$(dirname "$0")/../paper_1903_06631_b200/csrc"
make -s -j8 >/dev/null
F=$1; shift
B=${F%.cu}
mkdir -p ../ab build/ab
OBJS=$(ls build/*.o | grep -v "build/$B.o")
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
    -Xcompiler -fPIC -Xptxas -v -diag-suppress 177 $flags -c $F -o build/ab/${B}_$name.o \
    2> build/ab/$name.log || { cat build/ab/$name.log; exit 1; }
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../ab/lib_$name.so $OBJS \
    build/ab/${B}_$name.o -lcudart -lpthread
done
