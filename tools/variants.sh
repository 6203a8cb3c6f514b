#!/usr/bin/env bash
# Build compile-time variants of libgrape_walk.so into exp/ for A/B timing on the GPU.
#   tools/variants.sh NAME "-DFLAG=.. -DFLAG2=.." [NAME2 "FLAGS2" ...]
# Run one with: GRAPE_WALK_LIB=$PWD/exp/libgrape_walk_NAME.so python bench.py ...
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  objs=""
  for f in $(cd paper_2110_06196_b200/csrc && ls *.cu | sed 's/\.cu$//'); do
    nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v $flags \
         -c paper_2110_06196_b200/csrc/$f.cu -o build/${f}_$name.o 2> build/${f}_$name.ptxas.log
    objs="$objs build/${f}_$name.o"
  done
  nvcc $ARCH -shared -o exp/libgrape_walk_$name.so $objs -cudart static
  echo "built exp/libgrape_walk_$name.so ($flags)"
done
