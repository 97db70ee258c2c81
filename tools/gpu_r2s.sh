#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2s}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
for v in s0 s3 s4; do
  MPDE_LIB=$PWD/abtest/lib_$v.so timeout 900 python bench.py $A > $O/bench_$v.json 2> $O/bench_$v.err
done
ls -la $O
