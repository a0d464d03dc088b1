#!/bin/bash
# Build an A/B variant of the C-ABI library with extra compile definitions for one source:
#   bash tools/ab_variant.sh NAME SRC.cu [-DKNOB=V ...]   -> tools/ab_NAME.so
# (the other objects come from the in-tree build, paper_1308_6634_b200/_build)
set -e
NAME=$1; SRC=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_1308_6634_b200/_build
T=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off --expt-relaxed-constexpr "$@" -c $ROOT/paper_1308_6634_b200/csrc/$SRC -o $T/$SRC.o
objs=$(ls $B/*.o | grep -v "/$SRC.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/ab_$NAME.so $objs $T/$SRC.o -lcudart_static -lrt -lpthread -ldl
rm -rf $T
echo "built tools/ab_$NAME.so"
