#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2o}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf --timeout 600 -k "large_schur or vcycle" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
timeout 900 python bench.py $A > $O/bench_p1remap.json 2> $O/bench_p1remap.err
MPDE_P1_REMAP=0 timeout 900 python bench.py $A > $O/bench_nop1remap.json 2> $O/bench_nop1remap.err
ls -la $O
