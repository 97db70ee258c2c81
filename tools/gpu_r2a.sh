#!/bin/bash
# Round-2 session A: GPU suite, smoke, default bench line (C4 + C2/C3 sub-steps), tol_z sweep, C5 at N=1.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2a}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt; free -g >> $O/nproc.txt
timeout 1800 python -m pytest tests -m gpu -q -rf -x --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python tools/tolz_sweep.py 8 > $O/tolz.log 2>&1
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
ls -la $O
