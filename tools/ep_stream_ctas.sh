mkdir -p gpurun_out
for C in 4 8 16; do
FP8BS_EP_CTAS=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2963$((C % 10)) tests/ep_exchange_worker.py 65536 256 8 7168 2048 balanced > gpurun_out/exch2_ctas$C.json 2> gpurun_out/exch2_ctas$C.err; echo ctas=$C rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/exch2_ctas$C.json').read().strip().splitlines()[-1])
r=d['ranks'][0]; print({k:(round(v,3) if isinstance(v,float) else v) for k,v in r.items() if 'layer' in k or 'streamed' in k})"
done
