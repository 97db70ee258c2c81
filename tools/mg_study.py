"""MG preconditioner study: single-pass PCG iterations to a 1e-6 relative residual on NS
(C4-generator) problems, varying the V-cycle options.  Dev tool (GPU)."""
import os, sys, itertools, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from synth import gen
from paper_2502_18377_b200 import mpde

B = 4
shapes = [(16, 16, 16), (16, 32, 32), (32, 64, 64)]
for shape in shapes:
    gen.CONFIGS["X"] = gen.Config("X", 4, shape, (0.01, 1 / 64, 1 / 64), (0.0,) * 3, B, "ns2d")
    bt = synth.make_batch("X", batch=B)
    c = gu.to_dev(bt["c"]); b = gu.to_dev(bt["b"]); om = gu.to_dev(bt["omega"])
    grid = [dict()]
    grid += [dict(levels_max=L) for L in (2, 3)]
    grid += [dict(nu=n) for n in (1, 3, 4, 6)]
    grid += [dict(levels_max=2, nu=n) for n in (4, 8)]
    grid += [dict(smoother=0, nu=n) for n in (2, 4)]
    grid += [dict(cheb_ratio=r) for r in (8.0, 30.0, 120.0)]
    for kw in grid:
        if shape != (16, 16, 16) and kw.get("levels_max", 9) <= 2:
            continue
        o = mpde.mpde_default_options(tol_inner=1e-6, max_refine=1, tol_z=1e-12, tol=1e-12,
                                      max_iters=2000, **kw)
        s = mpde.Solver(shape, (0.01, 1 / 64, 1 / 64), c, opts=o)
        s.forward(b, om); torch.cuda.synchronize()
        st = s.stats_list(); s.close()
        print(shape, kw, "iters", [x["iters"] for x in st], "rel", ["%.1e" % x["rel_res"] for x in st],
              flush=True)
