#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/adapt3
mkdir -p $O
for T in "tol_adapt=0.1" "tol_adapt=0.1 tol_z=1.5e-5" "tol_adapt=0.1 tol_z=1e-5"; do
  for C in "C5 32" "C4 32" "C2 64" "C3 16"; do
    timeout 900 python tools/adapt_ref.py $C $T >> $O/ref.log 2>&1
  done
done
grep -h -A2 "opts=" $O/ref.log
