#!/bin/bash
# option sweep on the C4 step: poll interval, tol_z, tol_inner2
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2m}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
for o in "poll_every=8" "poll_every=4" "poll_every=2" "tol_z=1e-4" "tol_z=3e-5" "tol_z=1e-4 --opt poll_every=4"; do
  tag=$(echo $o | tr ' =-' '___')
  timeout 900 python bench.py $A --opt $o > $O/bench_$tag.json 2> $O/bench_$tag.err
done
ls -la $O
