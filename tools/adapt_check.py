"""Refinement-stop check on manufactured solutions (dev tool, GPU): per PDE the iterations,
refinement passes, the error estimate and the true relative error ||z - z_exact|| / ||z_exact||.

usage: [MPDE_TOL_ADAPT=..] python tools/adapt_check.py CONFIG B"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
cfg = synth.CONFIGS[name]
m = synth.make_mms(name, batch=B)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
s = mpde.Solver(cfg.shape, cfg.h, dev(m["c"]))
s.forward(dev(m["b"]), dev(m["omega"]))  # warm-up (graph capture)
torch.cuda.synchronize()
t0 = time.time()
z = s.forward(dev(m["b"]), dev(m["omega"]))
torch.cuda.synchronize()
t1 = time.time()
st = s.stats_list()
zz = z.cpu().numpy().astype(np.float64)
err = [float(np.linalg.norm(zz[i] - m["z_exact"][i]) / np.linalg.norm(m["z_exact"][i])) for i in range(B)]
its = [x["iters"] for x in st]
print(f"{name} B={B} MPDE_TOL_ADAPT={os.environ.get('MPDE_TOL_ADAPT', '-')}: fwd {1e3 * (t1 - t0):.0f} ms, "
      f"iters mean {np.mean(its):.1f} max {max(its)}, passes {sorted(set(x['refines'] for x in st))}, "
      f"max e_z {max(err):.2e}, max est {max(x['err_est'] for x in st):.2e}, "
      f"max e_z/est {max(e / max(x['err_est'], 1e-30) for e, x in zip(err, st)):.2f}")
print("  (iters, passes, est, e_z):", [(x["iters"], x["refines"], f"{x['err_est']:.1e}", f"{e:.1e}")
                                       for x, e in zip(st, err)])
s.close()
