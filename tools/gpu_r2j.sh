#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2j}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_dense.py -q -rf --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
timeout 900 python bench.py $A > $O/bench.json 2> $O/bench.err
MPDE_SMALL_FUSED=0 timeout 900 python bench.py $A > $O/bench_nosmallfused.json 2> $O/bench_nosmallfused.err
MPDE_SMALLP=8192 timeout 900 python bench.py $A > $O/bench_smallp8k.json 2> $O/bench_smallp8k.err
ls -la $O
