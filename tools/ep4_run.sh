set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_fullsize_gpu.py -k "balanced or split" tests/test_ep_exchange_gpu.py -q -x 2>&1 | tail -5
for P in balanced contiguous; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --placement $P > gpurun_out/n4_$P.json 2> gpurun_out/n4_$P.err; echo rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu --placement balanced > gpurun_out/n2_balanced.json 2> gpurun_out/n2_balanced.err; echo rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-c1 --no-pow2 > gpurun_out/n1_bal.json 2> gpurun_out/n1_bal.err; echo rc=$?
