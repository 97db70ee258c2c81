#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2d}
mkdir -p $O
timeout 600 python tools/march_check.py > $O/march_check.log 2>&1; echo "rc=$?" >> $O/march_check.log
timeout 900 python bench.py --no-cpu --no-subconfigs --no-fgmres --no-dense --no-template > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_schur_march" -s 4 -c 1 \
   -o $O/march_full python tools/prof_apply.py 2 > $O/ncu_full.log 2>&1
ls -la $O
