#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2r}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
timeout 900 python bench.py $A > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py $A > $O/bench2.json 2> $O/bench2.err
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -rf --timeout 600 -k "large_schur" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
ls -la $O
