#!/bin/bash
# Build variants of the device library that differ only in placement.cu
# compile flags, for A/B timing in one GPU call:
#   tools/ab_place.sh NAME:"-DFLAG=1" NAME2:"-DFLAG=0" ...
# -> paper_1903_06631_b200/ab/lib_NAME.so (load with MEMPLAN_LIB=...)
set -e
cd "$(dirname "$0")/../paper_1903_06631_b200/csrc"
make -s -j8 >/dev/null
mkdir -p ../ab build/ab
OBJS=$(ls build/*.o | grep -v placement.o)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
    -Xcompiler -fPIC -Xptxas -v -diag-suppress 177 $flags -c placement.cu -o build/ab/placement_$name.o \
    2> build/ab/$name.log || { cat build/ab/$name.log; exit 1; }
  grep -A3 "k_place_async" build/ab/$name.log | sed -n 3,4p | sed "s/^/$name: /"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../ab/lib_$name.so $OBJS \
    build/ab/placement_$name.o -lcudart -lpthread
done
