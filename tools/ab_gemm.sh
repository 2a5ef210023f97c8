#!/bin/bash
# A/B of GEMM builds in one GPU session (box-to-box variance is ~5%): for each library (in-tree "cur"
# or tools/libfp8bs_<name>.so) the C1 per-kernel numbers (bench.py --workload c1) and the C4 grouped
# anatomy (tools/grouped_anatomy.py).  Usage (on the GPU box): tools/ab_gemm.sh name...
for r in 1 2; do
for n in "$@"; do
  if [ "$n" = cur ]; then L=""; else L=tools/libfp8bs_$n.so; fi
  echo "== $n (round $r)"
  FP8BS_LIB=$L timeout 300 python bench.py --workload c1 --steps 20 --no-e2e --no-cpu --no-pow2 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  C1', {k:round(v['achieved']) for k,v in d['kernels'].items() if k.startswith('gemm')}, d['clocks']['sm_mhz'])"
  FP8BS_LIB=$L timeout 300 python tools/grouped_anatomy.py 7 | sed 's/^/  /'
done
done
