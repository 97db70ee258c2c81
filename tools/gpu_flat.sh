#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/flat
mkdir -p $O
for r in 1 2; do
  for v in 1 0; do MPDE_SMALL_FLAT=$v timeout 900 python bench.py --no-cpu > $O/bench_flat${v}_$r.json 2>&1; done
done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['c2_step']['value'],1), round(d['c3_step']['value'],1), {k: round(v['ms'],1) for k, v in d['kernels'].items() if k in ('schur_g','schur_out')})
"; done
timeout 1800 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_4d.py tests/test_gpu_golden.py tests/test_gpu_bc.py -q -rf --timeout 1200 -k "not variants_match_oracle_reference" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
