#!/bin/bash
# Runs on the GPU box (via gpurun): the default bench line, then ncu launch lists and --set full
# captures of the C4 grouped GEMM and of the C1 step's kernels.
# Usage: tools/gpu_bench_profile.sh <tag> [what=all|bench|ncu]
set -u
TAG=${1:-r02}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.csv 2>&1
free -g > $OUT/free_$TAG.txt 2>&1
if [ "$WHAT" != ncu ]; then
  timeout -s KILL 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
  tail -c 3000 $OUT/bench_$TAG.json
fi
[ "$WHAT" = bench ] && exit 0
C4="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-c1 --no-verify"
C1="python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-pow2"
timeout -s KILL 600 $C4 > $OUT/plain_c4_$TAG.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_quant|k_grouped|k_gemm' -c 2000 --csv \
    --log-file $OUT/launches_c4_$TAG.csv $C4 > $OUT/ncu_launches_c4_$TAG.log 2>&1; echo "ncu c4 launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_bs -s 3 -c 1 \
    -o $OUT/prof_grouped_$TAG $C4 > $OUT/ncu_grouped_$TAG.log 2>&1; echo "ncu grouped rc=$?"
timeout -s KILL 600 $C1 > $OUT/plain_c1_$TAG.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file $OUT/launches_c1_$TAG.csv $C1 > $OUT/ncu_launches_c1_$TAG.log 2>&1; echo "ncu c1 launches rc=$?"
# per C1 step: fprop, dgrad (full waves), dgrad (split-K tail), split-K reduce, wgrad; skip the 3 warm-up steps
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:'k_gemm_bs|k_splitk' -s 15 -c 5 \
    -o $OUT/prof_gemm_$TAG $C1 > $OUT/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_quant -s 9 -c 3 \
    -o $OUT/prof_quant_$TAG $C1 > $OUT/ncu_quant_$TAG.log 2>&1; echo "ncu quant rc=$?"
