#!/bin/bash
# Lanczos start-vector seed sensitivity of the C4 step (iteration tail), and tol_z 1e-4 vs 1e-5
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2l}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
for seed in 12345 1 777 31337 2024; do
  MPDE_LZ_SEED=$seed timeout 900 python bench.py $A > $O/bench_seed$seed.json 2> $O/bench_seed$seed.err
done
ls -la $O
