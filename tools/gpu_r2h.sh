#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2h}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
timeout 900 python bench.py $A > $O/bench_march.json 2> $O/bench_march.err
MPDE_PDL=0 timeout 900 python bench.py $A > $O/bench_march_nopdl.json 2> $O/bench_march_nopdl.err
MPDE_MARCH=0 timeout 900 python bench.py $A > $O/bench_twopass.json 2> $O/bench_twopass.err
MPDE_MARCH=0 MPDE_PDL=0 timeout 900 python bench.py $A > $O/bench_twopass_nopdl.json 2> $O/bench_twopass_nopdl.err
ls -la $O
