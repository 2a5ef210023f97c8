#!/bin/bash
# A/B of quantizer builds in one GPU session: tools/quant_bench.py (L2 flushed, each launch alone) and
# the in-step per-kernel GB/s of bench.py --workload c1.  Usage: tools/ab_quant.sh name...  (cur = in-tree)
for r in 1 2; do
for n in "$@"; do
  if [ "$n" = cur ]; then L=""; else L=tools/libfp8bs_$n.so; fi
  echo "== $n (round $r)"
  FP8BS_LIB=$L timeout 300 python tools/quant_bench.py 2>&1 | grep -i "dual\|weight" | sed 's/^/  /'
  FP8BS_LIB=$L timeout 300 python bench.py --workload c1 --steps 20 --no-e2e --no-cpu --no-pow2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  in-step', {k:round(v['achieved']) for k,v in d['kernels'].items() if not k.startswith('gemm')})"
done
done
