#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2g}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bc.py -q -rf -x --timeout 600 > $O/pytest_bc.log 2>&1; echo "rc=$?" >> $O/pytest_bc.log
timeout 900 python -m pytest tests/test_gpu_golden.py -q -rf -k C3 --timeout 600 > $O/pytest_golden.log 2>&1; echo "rc=$?" >> $O/pytest_golden.log
timeout 900 python bench.py --no-cpu --no-subconfigs --no-fgmres --no-dense --no-template > $O/bench_march.json 2> $O/bench_march.err
MPDE_MARCH=0 timeout 900 python bench.py --no-cpu --no-subconfigs --no-fgmres --no-dense --no-template > $O/bench_twopass.json 2> $O/bench_twopass.err
ls -la $O
