#!/usr/bin/env bash
# Build one compile-time variant of libgrape_walk.so into exp/, recompiling only walk_tab.cu
# (the other objects come from build/).   tools/variant1.sh NAME "-DFLAG=.."
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
ARCH="-gencode arch=compute_100a,code=sm_100a"
name=$1; flags=$2
nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Iinclude -Xptxas -v --expt-relaxed-constexpr $flags \
     -c paper_2110_06196_b200/csrc/walk_tab.cu -o build/walk_tab_$name.o 2> build/walk_tab_$name.ptxas.log
objs=$(ls build/*.o | grep -v "_[a-z0-9]*\.o$\|walk_tab" || true)
nvcc $ARCH -shared -o exp/libgrape_walk_$name.so build/capi.o build/dist.o build/graph.o build/graph_tables.o \
     build/partition.o build/skipgram.o build/walk.o build/walk_cdf.o build/walk_sm.o build/walk_tab_$name.o -cudart static
grep -A2 "ILb1ELb1ELb0ELb1ELb1ELb0ELi0ELb0" build/walk_tab_$name.ptxas.log | grep -i "registers\|spill" | head -2
echo "built exp/libgrape_walk_$name.so ($flags)"
