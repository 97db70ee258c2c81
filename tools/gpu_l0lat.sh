#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/l0lat
mkdir -p $O
for r in 1 2; do
  for v in 0 1; do MPDE_L0_LAT=$v timeout 900 python bench.py --no-cpu > $O/bench_l0lat${v}_$r.json 2>&1; done
done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['schur_g_l0']['frac'],4), round(d['c3_step']['value'],1), d['iters']['fwd_mean'])
"; done
MPDE_L0_LAT=1 timeout 900 python -m pytest tests/test_gpu_golden.py -q -k "full_size_matches" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
