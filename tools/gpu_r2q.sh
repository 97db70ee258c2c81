#!/bin/bash
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2q}
mkdir -p $O
A="--no-cpu --no-subconfigs --no-fgmres --no-dense --no-template --no-e2e --steps 3"
for c in 0 16 8 4; do
  MPDE_L0_CHUNK=$c timeout 900 python bench.py $A > $O/bench_chunk$c.json 2> $O/bench_chunk$c.err
done
MPDE_L0_CHUNK=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -rf --timeout 900 > $O/pytest_chunk8.log 2>&1; echo "rc=$?" >> $O/pytest_chunk8.log
ls -la $O
