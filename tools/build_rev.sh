#!/bin/bash
# Build libnnt.so of a git revision into abtest/<rev>/libnnt.so (A/B kernel timing).
#   tools/build_rev.sh <rev>
set -e
REV=$1
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/abtest/$REV
rm -rf $OUT && mkdir -p $OUT/src
git -C $ROOT archive $REV paper_2504_13236_b200/csrc include | tar -x -C $OUT/src
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -I $OUT/src/include -DNDEBUG"
objs=""
for f in $OUT/src/paper_2504_13236_b200/csrc/*.cu $OUT/src/paper_2504_13236_b200/csrc/*.cpp; do
  o=$OUT/$(basename $f).o; $NVCC $FLAGS -c $f -o $o & objs="$objs $o"
done
wait
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libnnt.so $objs
echo $OUT/libnnt.so
