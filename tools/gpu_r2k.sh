#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2k}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -rf --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
timeout 900 python bench.py $A > $O/bench.json 2> $O/bench.err
MPDE_SLAB=0 timeout 900 python bench.py $A > $O/bench_noslab.json 2> $O/bench_noslab.err
timeout 900 python bench.py --config C3 --no-cpu --no-e2e --steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
MPDE_SLAB=0 timeout 900 python bench.py --config C3 --no-cpu --no-e2e --steps 3 > $O/bench_c3_noslab.json 2> $O/bench_c3_noslab.err
ls -la $O
