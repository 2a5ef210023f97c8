set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_scatter_gpu.py tests/test_ep_exchange_gpu.py -q -x 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29610 tests/ep_exchange_worker.py 65536 256 8 7168 2048 balanced > gpurun_out/exch4_fused.json 2> gpurun_out/exch4_fused.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-c1 > gpurun_out/n4_fused.json 2> gpurun_out/n4_fused.err; echo rc=$?
