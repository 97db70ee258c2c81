#!/bin/bash
# y edge rows in shared memory (pass 2), natural quad mapping default: parity + bench + ncu.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/yedge
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_golden.py -q -rf --timeout 1200 -k "not variants_match_oracle_reference" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 900 python bench.py --no-cpu > $O/bench_$r.json 2>&1; done
for f in $O/bench_*.json; do python -c "
import json
d=json.loads([l for l in open('$f').read().splitlines() if l.startswith('{')][-1])
print('$f', round(d['value'],2), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],2), round(d['schur_g_l0']['frac'],4), d['iters']['fwd_mean'], d['clocks']['sm_mhz'], d['c2_step']['value'], d['c3_step']['value'])
"; done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_schur_s_b22" -s 49 -c 1 -o $O/b22 python tools/prof_step.py 1 > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/b22.ncu-rep $O/ncu_b22.txt "(C4 level 0 pass 2, natural mapping, y edge rows in smem)" > /dev/null 2>&1
cat $O/ncu_b22.txt; tail -3 $O/pytest.log
