#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/s5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fgmres.py tests/test_gpu_dense.py -x -q -s > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/pytest_new.log
timeout 600 python tools/fgmres_sweep.py 0 20 30 32 > $O/sweep.log 2>&1
MPDE_GM_REORTH=0 timeout 300 python tools/fgmres_sweep.py 30 >> $O/sweep.log 2>&1
