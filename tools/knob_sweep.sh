#!/bin/bash
# One GPU session: default bench line (PCG) under each existing schur.cu / mpde.cu env knob.
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/${TAG:-knobs}
mkdir -p $O
F="--no-e2e --no-cpu --no-template --no-dense --no-fgmres --steps 5 --warmup 3"
for kv in "X=0" "MPDE_HY=1" "MPDE_SMALLP=4096" "MPDE_SMALLP=65536" "MPDE_SCHUR_BLOCK=2" "MPDE_PDL=0" "MPDE_B22_TP=2" "X=1"; do
  echo -n "$kv " >> $O/knobs.log
  env $kv timeout 300 python bench.py $F 2>>$O/knobs.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['ms_per_step'],2), d['iters']['fwd_mean'], d['iters']['bwd_mean'], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/knobs.log 2>&1
done
