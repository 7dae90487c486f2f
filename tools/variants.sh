#!/bin/bash
# Builds kernel variants of libsfem_b200.so into variants/<name>.so for A/B
# timing on the GPU box (SFEM_LIB=variants/<name>.so python tools/kernel_times.py).
#   tools/variants.sh name "-DFLAG=1 ..." [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/../paper_1701_03967_b200"
mkdir -p ../variants
while [ $# -ge 2 ]; do
  (make -j16 BUILD=../variants/$1.build OUT=../variants/$1.so EXTRA="$2" > ../variants/$1.log 2>&1 && rm -rf ../variants/$1.build) &
  shift 2
done
wait
