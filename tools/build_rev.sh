#!/bin/bash
# Build libfp8bs.so from a git revision into tools/libfp8bs_<name>.so (A/B experiments; optional
# extra nvcc flags, e.g. -DFP8BS_GEMM_TRACE=1).  Usage: tools/build_rev.sh <rev|WORKTREE> <name> [nvcc flags...]
set -e
REV=$1; NAME=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p $TMP/p/csrc $TMP/include   # mirrors the repo layout (api.cu includes ../../include/fp8bs.h)
if [ "$REV" = WORKTREE ]; then
  cp $ROOT/paper_2412_19437_b200/csrc/* $TMP/p/csrc/; cp $ROOT/include/fp8bs.h $TMP/include/
else
  for f in $(git -C $ROOT ls-tree --name-only $REV paper_2412_19437_b200/csrc/); do git -C $ROOT show $REV:$f > $TMP/p/csrc/$(basename $f); done
  git -C $ROOT show $REV:include/fp8bs.h > $TMP/include/fp8bs.h
fi
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -prec-div=true -prec-sqrt=true -ftz=false -fmad=true -Xcompiler -fPIC,-O2,-fvisibility=hidden -cudart static --expt-relaxed-constexpr"
for f in $TMP/p/csrc/*.cu; do nvcc $FLAGS "$@" -I $TMP/include -c $f -o $f.o & done; wait
for f in $TMP/p/csrc/*.cu; do [ -f $f.o ] || { echo "build failed: $f"; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o $ROOT/tools/libfp8bs_$NAME.so $TMP/p/csrc/*.o -lpthread -ldl -lrt
rm -rf $TMP
echo $ROOT/tools/libfp8bs_$NAME.so
