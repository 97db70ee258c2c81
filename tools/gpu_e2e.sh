#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/e2e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "host_abi or fwd_bwd_random" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 900 python bench.py --no-cpu > $O/bench_$r.json 2>&1; done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['e2e']['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])
"; done
tail -2 $O/pytest.log
