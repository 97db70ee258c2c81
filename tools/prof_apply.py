"""One hierarchy at C4 size (32 PDEs, (32,64,64)) and a few S applies / V-cycles on level 0:
the workload ncu captures for the S-apply kernels (tools/gpu_*.sh)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2502_18377_b200 import mpde
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
bt = synth.make_batch("C4", 32)
cfg = bt["cfg"]
s = mpde.Solver(cfg.shape, cfg.h, torch.from_numpy(bt["c"]).cuda())
x = torch.randn((32, cfg.shape[0] * cfg.shape[1] * cfg.shape[2]), device="cuda")
y = torch.empty_like(x)
for _ in range(n):
    mpde.mpde_apply_schur(s.h_, 0, x, y)
    mpde.mpde_apply_precond(s.h_, x, y)
torch.cuda.synchronize()
print("ok")
