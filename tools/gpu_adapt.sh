#!/bin/bash
# Adaptive pass-3 tolerance A/B (MPDE_TOL_ADAPT): MMS true errors vs estimates, golden parity,
# bench lines C4 / C5.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/adapt
mkdir -p $O
for A in 0 0.05 0.1 0.3; do
  for C in "C5 16" "C4 32" "C3 16" "C2 64"; do
    MPDE_TOL_ADAPT=$A timeout 600 python tools/adapt_check.py $C >> $O/mms.log 2>&1
  done
done
MPDE_TOL_ADAPT=0.1 timeout 1800 python -m pytest tests/test_gpu_golden.py -q -rf --timeout 1200 > $O/golden_01.log 2>&1; echo "rc=$?" >> $O/golden_01.log
MPDE_TOL_ADAPT=0.1 timeout 900 python bench.py --no-cpu > $O/bench_c4_01.json 2>&1
MPDE_TOL_ADAPT=0.1 timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > $O/bench_c5_01.json 2>&1
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > $O/bench_c5_0.json 2>&1
grep -h "MPDE_TOL_ADAPT" $O/mms.log
