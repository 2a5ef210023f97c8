#!/bin/bash
# Expert-parallel scaling of the grouped expert GEMM (BASELINE configs[4]) on one box:
# bench.py --workload c4 at N = 1, 2, 4 (, 8) GPUs, one JSON line each -> gpurun_out/ep_<tag>_N<n>.json
# Usage (on the GPU box): tools/ep_scaling.sh <tag> [max_gpus]
# (setsid: torchrun signals its whole process group on exit, which would end this script)
set -u
TAG=${1:-r01}; MAX=${2:-4}
mkdir -p gpurun_out
for n in 1 2 4 8; do
  [ $n -gt $MAX ] && break
  if [ $n -eq 1 ]; then
    timeout -s KILL 900 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu --no-c1 --no-e2e > gpurun_out/ep_${TAG}_N$n.json 2> gpurun_out/ep_${TAG}_N$n.err
  else
    setsid timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n --workload c4 --steps 20 --warmup 3 --no-cpu --no-c1 --no-e2e \
      > gpurun_out/ep_${TAG}_N$n.json 2> gpurun_out/ep_${TAG}_N$n.err
  fi
  echo "N=$n rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/ep_${TAG}_N$n.json').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['ep'], d['clocks'])" 2>&1 | tail -1)"
done
