#!/bin/bash
# full GPU suite, per-kernel ncu table (C4 step), small-case driver
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2i}
mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/kernels.csv python tools/prof_step.py 1 > $O/ncu_kernels.log 2>&1
python tools/kernel_table.py $O/kernels.csv $O/kernel_table.txt > /dev/null 2>&1
# compute-sanitizer is closed on this GPU pool; the small-case driver runs plainly instead
timeout 600 python tools/sanitize_case.py > $O/small_cases.log 2>&1; echo "rc=$?" >> $O/small_cases.log
MPDE_MARCH=2 timeout 600 python tools/sanitize_case.py > $O/small_cases_march.log 2>&1; echo "rc=$?" >> $O/small_cases_march.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
ls -la $O
