mkdir -p gpurun_out
FP8BS_EP_CTAS=16 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/ep_exchange_worker.py 65536 256 8 7168 2048 balanced > gpurun_out/exch2_disp.json 2> gpurun_out/exch2_disp.err; echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/exch2_disp.json').read().strip().splitlines()[-1])
r=d['ranks'][0]; print({k:(round(v,3) if isinstance(v,float) else v) for k,v in r.items() if 'ms' in k or 'streamed' in k})"
tail -3 gpurun_out/exch2_disp.err
