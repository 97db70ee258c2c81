#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2n}
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_bc.py tests/test_gpu_multirank.py tests/test_gpu_golden.py -q -rf --timeout 900 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
ls -la $O
