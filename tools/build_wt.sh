#!/bin/bash
# Build libnnt.so of the WORKING TREE with extra nvcc flags into abtest/<name>/libnnt.so (A/B timing).
#   tools/build_wt.sh <name> [-DFLAG ...]
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/abtest/$NAME
rm -rf $OUT && mkdir -p $OUT
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $ROOT/include -DNDEBUG $*"
objs=""
for f in $ROOT/paper_2504_13236_b200/csrc/*.cu $ROOT/paper_2504_13236_b200/csrc/*.cpp; do
  o=$OUT/$(basename $f).o; $NVCC $FLAGS -c $f -o $o & objs="$objs $o"
done
wait
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libnnt.so $objs
echo $OUT/libnnt.so
