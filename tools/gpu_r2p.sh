#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2p}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_golden.py -q -rf --timeout 900 > $O/pytest_golden.log 2>&1; echo "rc=$?" >> $O/pytest_golden.log
timeout 1200 python tools/tolz_golden.py > $O/tolz_golden.log 2>&1; echo "rc=$?" >> $O/tolz_golden.log
ls -la $O
