"""C5 (64,128,128) forward iteration counts per PDE under option / env variants (dev tool, GPU).

usage: python tools/c5_iters.py B [key=value ...]   (mpde_options fields)
Prints per-PDE (iters, refines, err_est) and the lambda_max estimates of level 0."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

B = int(sys.argv[1])
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = float(v) if "." in v or "e" in v else int(v)
cfg = synth.CONFIGS["C5"]
bt = synth.make_batch("C5", batch=B)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]), opts=mpde.mpde_default_options(**kw))
lm = torch.empty(B, dtype=torch.float32, device="cuda")
mpde.mpde_hierarchy_query(s.h_, 0, 2, lm)
torch.cuda.synchronize()
t0 = time.time()
z = s.forward(dev(bt["b"]), dev(bt["omega"]))
torch.cuda.synchronize()
t1 = time.time()
st = s.stats_list()
its = [x["iters"] for x in st]
print(f"env LZ_SEED={os.environ.get('MPDE_LZ_SEED', '-')} opts={kw}: fwd {1e3 * (t1 - t0):.0f} ms, iters mean "
      f"{np.mean(its):.1f} max {max(its)}; refines {sorted(set(x['refines'] for x in st))}")
print("  per PDE (iters, refines, err_est):", [(x["iters"], x["refines"], f"{x['err_est']:.1e}") for x in st])
print("  lambda_max l0:", np.round(lm.cpu().numpy(), 3).tolist())
s.close()
