#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2c}
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_schur_march" -s 2 -c 3 \
   -o $O/march_full python tools/prof_apply.py 2 > $O/ncu_full.log 2>&1
timeout 600 env MPDE_MARCH=0 ncu --set full --clock-control none -k "regex:k_schur_(s_b22|h_v4)" -s 4 -c 2 \
   -o $O/twopass_full python tools/prof_apply.py 2 > $O/ncu_full2.log 2>&1
ls -la $O
