#!/bin/bash
# C5 iteration-count A/B: HEAD library vs the b5577ba build (abtest/), 32 distinct PDEs.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/c5ab
mkdir -p $O
for L in paper_2502_18377_b200/libmpde.so abtest/libmpde_b5577ba.so; do
  echo "== $L" >> $O/c5.log
  MPDE_LIB=$PWD/$L timeout 600 python tools/c5_iters.py 32 >> $O/c5.log 2>&1
done
MPDE_LZ_SEED=777 timeout 600 python tools/c5_iters.py 32 >> $O/c5.log 2>&1
timeout 600 python tools/c5_iters.py 32 lanczos_steps=24 >> $O/c5.log 2>&1
cat $O/c5.log
