mkdir -p gpurun_out
for N in 2 4; do
T0=$(date +%s)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2967$N bench.py --gpus $N > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err; echo N=$N rc=$? wall $(( $(date +%s) - T0 )) s
done
