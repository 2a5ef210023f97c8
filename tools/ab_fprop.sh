#!/bin/bash
# A/B of the GEMM against tools/libfp8bs_prev.so (experiments only).  Usage: tools/ab_fprop.sh tag [cases]
set -u
mkdir -p gpurun_out
OUT=gpurun_out/ab_${1:-x}.txt
CASES=${2:-fprop}
: > $OUT
timeout 200 python tools/gemm_matrix.py 2,1 0 $CASES 2>&1 | sed "s/^/new /" | tee -a $OUT
FP8BS_LIB=tools/libfp8bs_prev.so timeout 200 python tools/gemm_matrix.py ${PREV_VARIANTS:-2,1} 0 $CASES 2>&1 | sed "s/^/old /" | tee -a $OUT
