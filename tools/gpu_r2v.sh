#!/bin/bash
# Round-2 verification session: 4D parity tests, the parity tests touching the query ABI, the
# default bench line (slab-based CPU baseline) and the reference arm.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2v}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_4d.py -q -rf --timeout 1200 -s > $O/pytest_4d.log 2>&1; echo "pytest rc=$?" >> $O/pytest_4d.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
ls -la $O
