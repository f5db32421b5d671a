#!/bin/bash
# build an experimental variant of the library: tools/build_variant.sh NAME "-DMACRO=V ..."
# -> build_ab/NAME.so (load it with FT_LIB=build_ab/NAME.so)
set -e
cd "$(dirname "$0")/../paper_1804_09152_b200/csrc"
mkdir -p ../../build_ab/$1
for f in *.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC \
       -I../../include $2 -Xptxas -v -c $f -o ../../build_ab/$1/${f%.cu}.o 2> ../../build_ab/$1/${f%.cu}.ptxas.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build_ab/$1.so ../../build_ab/$1/*.o -lcudart
