#!/bin/bash
# FFMA2 quad updates A/B (abtest/libmpde_scalar.so = the scalar form), parity of the variants.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ffma2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -q -rf --timeout 1200 -k "not variants_match_oracle_reference" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  timeout 900 python bench.py --no-cpu > $O/bench_ffma2_$r.json 2>&1
  MPDE_LIB=$PWD/abtest/libmpde_scalar.so timeout 900 python bench.py --no-cpu > $O/bench_scalar_$r.json 2>&1
done
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), round(d['schur_g_l0']['frac'],4) if 'schur_g_l0' in d else '', d['iters']['fwd_mean'], d['clocks']['sm_mhz'])
"; done
tail -3 $O/pytest.log
