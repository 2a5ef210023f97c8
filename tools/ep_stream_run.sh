set -x
mkdir -p gpurun_out
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29620 tests/ep_exchange_worker.py > gpurun_out/exch2_stream_small.json 2> gpurun_out/exch2_stream_small.err; echo rc=$?
tail -3 gpurun_out/exch2_stream_small.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tests/ep_exchange_worker.py 65536 256 8 7168 2048 balanced > gpurun_out/exch2_stream_c4.json 2> gpurun_out/exch2_stream_c4.err; echo rc=$?
tail -3 gpurun_out/exch2_stream_c4.err
