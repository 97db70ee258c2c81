#!/bin/bash
# Round-2 final session (after the adaptive last pass / tol_z 1.5e-5 defaults): GPU suite, smoke,
# default bench line (C4 + C2/C3 sub-steps), C5 line.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2final2}
mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -rf --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
ls -la $O
