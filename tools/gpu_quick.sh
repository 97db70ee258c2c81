#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-q}
mkdir -p $O
timeout 600 python tools/march_check.py > $O/march_check.log 2>&1; echo "rc=$?" >> $O/march_check.log
