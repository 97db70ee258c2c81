"""Is the derivative-field error of the manufactured C4 adjoint test an input-rounding floor?
Solve with default and with much tighter settings; a floor does not move.  Dev tool (GPU)."""
import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from oracle import Problem, assemble, normal_apply
from paper_2502_18377_b200 import mpde
m = synth.make_mms("C4", batch=2)
cfg = m["cfg"]; pr = Problem(cfg.shape, cfg.h); P = int(np.prod(cfg.shape))
g = np.zeros((2, 7, P), np.float32)
for i in range(2):
    A, _, _ = assemble(pr, m["c"][i].astype(np.float64), m["b"][i].astype(np.float64), m["omega"][i].astype(np.float64))
    g[i] = normal_apply(A, m["z_exact"][i].reshape(-1)).reshape(7, P).astype(np.float32)
for kw in ({}, dict(tol=1e-12, tol_z=1e-10, tol_inner=1e-6, max_refine=12, precision=3)):
    out = gu.gpu_solve(cfg.shape, cfg.h, m["c"], m["b"], m["omega"], g, opts=mpde.mpde_default_options(**kw), want_dz=True)
    print(kw, [("%.2e" % gu.rel(out["dz"][i][0], m["z_exact"][i][0]), "%.2e" % gu.rel(out["dz"][i], m["z_exact"][i]),
                [s["iters"] for s in out["stats_bwd"]][i]) for i in range(2)], flush=True)
