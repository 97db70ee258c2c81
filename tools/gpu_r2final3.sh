#!/bin/bash
# Round-2 final session: GPU suite, smoke, default bench line, C5 line, launch list, ncu full
# capture of the level-0 S kernels.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-r2final3}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q -rf --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 1500 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python tools/prof_step.py 2 > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches.csv $O/launches_summary.txt "round 2 final" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_schur_(s_b22|h_v4)" -s 98 -c 2 \
   -o $O/l0_full python tools/prof_step.py 1 > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/l0_full.ncu-rep $O/ncu_l0_summary.txt "(C4 level 0, one pass-1 and one pass-2 launch)" > /dev/null 2>&1

# keep the merge under gpurun's 64 MiB: the summaries above carry what is judged
rm -f $O/l0_full.ncu-rep; gzip -f $O/launches.csv
ls -la $O
