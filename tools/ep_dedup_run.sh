mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ep_exchange_gpu.py -q -x 2>&1 | tail -3
for N in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2965$N tests/ep_exchange_worker.py 65536 256 8 7168 2048 balanced > gpurun_out/exch${N}_dedup.json 2> gpurun_out/exch${N}_dedup.err; echo N=$N rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/exch${N}_dedup.json').read().strip().splitlines()[-1])
r=d['ranks'][0]; print({k:(round(v,3) if isinstance(v,float) else v) for k,v in r.items() if 'ms' in k or 'bitwise' in k})"
done
