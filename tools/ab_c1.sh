# same-box A/B of the C1 step's per-kernel numbers: tools/ab_c1.sh libA libB [rounds]
for i in $(seq 1 ${3:-2}); do for L in "$1" "$2"; do
  FP8BS_LIB=$L timeout 300 python bench.py --workload c1 --no-e2e --no-cpu --no-pow2 > gpurun_out/abc1.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/abc1.json').read().strip().splitlines()[-1])
k=d['kernels']; print('$L'.split('/')[-1], round(d['value']), {n:(round(v['ms']*1e3,1), round(v['achieved'])) for n,v in k.items()}, d['clocks']['sm_mhz'])"
done; done
