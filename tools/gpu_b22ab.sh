#!/bin/bash
# pass-2 register / y-window A/B (abtest/ builds): default, streamed y window, 4 CTAs/SM.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/b22ab
mkdir -p $O
for r in 1 2; do
  timeout 900 python bench.py --no-cpu > $O/bench_default_$r.json 2>&1
  for v in ys1_mb3 ys1_mb4 ys0_mb4; do
    MPDE_LIB=$PWD/abtest/libmpde_$v.so timeout 900 python bench.py --no-cpu > $O/bench_${v}_$r.json 2>&1
  done
done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), round(d['schur_g_l0']['frac'],4), d['iters']['fwd_mean'], d['clocks']['sm_mhz'], round(d['c2_step']['value'],1), round(d['c3_step']['value'],1))
"; done
