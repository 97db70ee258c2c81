#!/bin/bash
# Round-2 session B: march kernel check, kernel tests, bench.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2b}
mkdir -p $O
timeout 600 python tools/march_check.py > $O/march_check.log 2>&1; echo "rc=$?" >> $O/march_check.log
timeout 1200 python -m pytest tests/test_gpu_kernels.py -q -rf --timeout 600 > $O/pytest_kernels.log 2>&1; echo "pytest rc=$?" >> $O/pytest_kernels.log
timeout 900 python bench.py --no-cpu --no-subconfigs --no-fgmres --no-dense > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
ls -la $O
