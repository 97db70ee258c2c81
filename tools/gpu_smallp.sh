#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/smallp
mkdir -p $O
for v in 16384 8192 16384 8192; do
  MPDE_SMALLP=$v timeout 900 python bench.py --no-cpu > $O/bench_$v_$RANDOM.json 2>&1
done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['c2_step']['value'],1), round(d['c3_step']['value'],1), {k: round(v['ms'],1) for k, v in d['kernels'].items() if v['ms'] > 0})
"; done
