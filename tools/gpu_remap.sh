#!/bin/bash
# Quad mapping A/B: warp-specialised interior/edge remap (default) vs natural row-contiguous.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/remap
mkdir -p $O
for r in 1 2; do
  timeout 900 python bench.py --no-cpu > $O/bench_remap1_$r.json 2>&1
  MPDE_REMAP=0 timeout 900 python bench.py --no-cpu > $O/bench_remap0_$r.json 2>&1
done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), round(d['schur_g_l0']['frac'],4), d['iters']['fwd_mean'], d['clocks']['sm_mhz'], d['c2_step']['value'], d['c3_step']['value'])
"; done
MPDE_REMAP=0 timeout 900 ncu --set full --clock-control none -k "regex:k_schur_s_b22" -s 49 -c 1 -o $O/b22_remap0 python tools/prof_step.py 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/b22_remap0.ncu-rep $O/ncu_remap0.txt "(C4 level 0 pass 2, MPDE_REMAP=0)" > /dev/null 2>&1
cat $O/ncu_remap0.txt
