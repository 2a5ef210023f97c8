#!/bin/bash
# Runs on the GPU box (via gpurun): bench line, then ncu launch list + full captures.
# Usage: tools/gpu_bench_profile.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.csv 2>&1
timeout -s KILL 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json
PROF="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 600 $PROF > $OUT/plain_$TAG.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file $OUT/launches_$TAG.csv $PROF > $OUT/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm_bs -s 9 -c 3 \
    -o $OUT/prof_gemm_$TAG $PROF > $OUT/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_quant -s 9 -c 3 \
    -o $OUT/prof_quant_$TAG $PROF > $OUT/ncu_quant_$TAG.log 2>&1; echo "ncu quant rc=$?"
