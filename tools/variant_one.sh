#!/bin/bash
# Variant of libsfem_b200.so that recompiles ONE translation unit with extra
# flags and links it with the in-tree objects (seconds instead of minutes):
#   tools/variant_one.sh <name> <unit (e.g. sweep_rows)> "<flags>"
# -> variants/<name>.so ; run with SFEM_LIB=variants/<name>.so
set -e
cd "$(dirname "$0")/../paper_1701_03967_b200"
name=$1; unit=$2; flags=$3
mkdir -p ../variants/$name.build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 -Xptxas -v $flags \
  -c csrc/$unit.cu -o ../variants/$name.build/$unit.o 2> ../variants/$name.ptxas
objs=$(ls build/*.o | grep -v "build/$unit.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../variants/$name.so $objs ../variants/$name.build/$unit.o -lgomp
rm -rf ../variants/$name.build
echo "built variants/$name.so"
