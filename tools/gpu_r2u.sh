#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2u}
mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_golden.py "tests/test_gpu_parity.py::test_mms_full_size" -q -rf -s --timeout 1200 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
ls -la $O
