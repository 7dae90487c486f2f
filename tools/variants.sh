#!/bin/bash
# Builds kernel variants of libsfem_b200.so into variants/<name>.so for A/B
# timing on the GPU box (SFEM_LIB=variants/<name>.so python tools/kernel_times.py).
#   tools/variants.sh name "-DFLAG=1 ..." [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/../paper_1701_03967_b200"
mkdir -p ../variants
while [ $# -ge 2 ]; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-fopenmp,-O3 $2 -shared -o ../variants/$1.so \
    csrc/*.cu csrc/*.cpp -lgomp > ../variants/$1.log 2>&1 &
  shift 2
done
wait
