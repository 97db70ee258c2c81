#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/adapt2
mkdir -p $O
for A in 0 0.1 0.3; do
  for C in "C5 32" "C4 32" "C2 64" "C3 16"; do
    MPDE_TOL_ADAPT=$A timeout 900 python tools/adapt_ref.py $C >> $O/ref.log 2>&1
  done
done
grep -h -A1 "MPDE_TOL_ADAPT" $O/ref.log
