#!/bin/bash
# A/B/C... of GEMM builds: tools/ab_multi.sh <cases> <variant> <name>... (name "cur" = the in-tree library,
# others tools/libfp8bs_<name>.so).  Experiments only.
set -u
CASES=$1; V=$2; shift 2
for n in "$@"; do
  if [ "$n" = cur ]; then L=""; else L=tools/libfp8bs_$n.so; fi
  FP8BS_LIB=$L timeout 200 python tools/gemm_matrix.py $V 0 $CASES 2>&1 | sed "s/^/$n /"
done
