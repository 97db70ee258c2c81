#!/bin/bash
# GPU session: new tests (FGMRES, dense path) and the bench line with the new sub-steps.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-s4}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fgmres.py tests/test_gpu_dense.py -x -q -s > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/pytest_new.log
timeout 900 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
