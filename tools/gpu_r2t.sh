#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2t}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
for v in h5 h6 h5b h6b; do
  lib=${v%b}
  MPDE_LIB=$PWD/abtest/lib_$lib.so timeout 900 python bench.py $A > $O/bench_$v.json 2> $O/bench_$v.err
done
ls -la $O
