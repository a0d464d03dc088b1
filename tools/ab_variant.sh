#!/bin/bash
# Build an A/B variant of the C-ABI library with extra compile definitions for one source:
#   bash tools/ab_variant.sh NAME SRC.cu [-DKNOB=V ...]   -> tools/ab_NAME.so
#   bash tools/ab_variant.sh NAME REV:SRC.cu [...]        -> the same source (and its headers) at git REV
# (the other objects come from the in-tree build, paper_1308_6634_b200/_build)
set -e
NAME=$1; SRC=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=$ROOT/paper_1308_6634_b200/_build
T=$(mktemp -d)
DIR=$ROOT/paper_1308_6634_b200/csrc
if [[ "$SRC" == *:* ]]; then  # sources of another revision
  REV=${SRC%%:*}; SRC=${SRC#*:}
  mkdir -p $T/a/b/src $T/a/include && git -C $ROOT show $REV:include/mlsqr_b200.h > $T/a/include/mlsqr_b200.h
  for f in $(git -C $ROOT ls-tree --name-only $REV paper_1308_6634_b200/csrc/); do
    git -C $ROOT show $REV:$f > $T/a/b/src/$(basename $f)
  done
  DIR=$T/a/b/src
fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off --expt-relaxed-constexpr "$@" -I$ROOT/include -c $DIR/$SRC -o $T/$SRC.o
objs=$(ls $B/*.o | grep -v "/$SRC.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/ab_$NAME.so $objs $T/$SRC.o -lcudart_static -lrt -lpthread -ldl
rm -rf $T
echo "built tools/ab_$NAME.so"
