#!/bin/bash
# One GPU session: parity suite, smoke, default bench line, launch list, ncu full capture of level-0 S pass 2.
set -x
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-s3}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python tools/prof_step.py 2 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_schur_(s_b22|h_v4)" -s 98 -c 2 \
   -o $O/l0_full python tools/prof_step.py 1 > $O/ncu_full.log 2>&1
timeout 400 python tools/fgmres_sweep.py 0 30 > $O/sweep.log 2>&1
ls -la $O
