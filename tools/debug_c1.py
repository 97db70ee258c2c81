import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth, gpu_util as gu
from oracle import Problem, solve_forward, solve_backward
from paper_2502_18377_b200 import mpde
bt = synth.make_batch("C1"); cfg = bt["cfg"]; g = synth.make_g("C1")
pr = Problem(cfg.shape, cfg.h)
f = solve_forward(pr, bt["c"][0], bt["b"][0], bt["omega"][0], method="dense")
bw = solve_backward(pr, f, g[0].reshape(-1).astype(np.float64), method="dense")
for kw in ({}, {"levels_max": 1}, {"tol": 1e-9}, {"tol": 1e-10, "max_refine": 8}):
    out = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g, opts=mpde.mpde_default_options(**kw))
    print(kw, "z norm", np.linalg.norm(out["z"]), "ez", gu.rel(out["z"][0], f["z"]), [gu.rel(out[k][0], bw[k]) for k in ("grad_c","grad_b","grad_omega")], out["stats_fwd"], out["stats_bwd"])
rng = np.random.default_rng(31)
shape=(16,16); h=(1/15,1/15); B=2
c = rng.normal(0.0, 0.5, (B, 5, 256)); c[:, 1] += 1.0
b = rng.normal(size=(B, 256)); om = rng.normal(size=(B, 256)); gg = rng.normal(size=(B, 5, 256))
c,b,om,gg=[a.astype(np.float32) for a in (c,b,om,gg)]
w=(1.25,2.0,0.75,0.875)
pr = Problem(shape, h, *w)
f = solve_forward(pr, c[0], b[0], om[0], method="dense")
bw = solve_backward(pr, f, gg[0].reshape(-1).astype(np.float64), method="dense")
for kw in ({}, {"tol": 1e-9}, {"tol": 1e-10, "max_refine": 8}, {"tol":1e-12,"max_refine":10}):
    out = gu.gpu_solve(shape, h, c, b, om, gg, weights=w, opts=mpde.mpde_default_options(**kw))
    print(kw, "ez", gu.rel(out["z"][0], f["z"]), [gu.rel(out[k][0], bw[k]) for k in ("grad_c","grad_b","grad_omega")], "dz", gu.rel(out["dz"][0], bw["dz"]), out["stats_fwd"][0], out["stats_bwd"][0])
