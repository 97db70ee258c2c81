import sys, os, time, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth, gpu_util as gu
from paper_2502_18377_b200 import mpde
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = synth.make_mms(name, batch=B); cfg = m["cfg"]
for kw in ({}, {"tol_inner": 1e-5}, {"nu": 3}, {"smoother": 0}, {"max_refine": 8, "tol": 1e-9}):
    torch.cuda.synchronize(); t = time.time()
    out = gu.gpu_solve(cfg.shape, cfg.h, m["c"], m["b"], m["omega"], opts=mpde.mpde_default_options(**kw))
    dt = time.time() - t
    errs = [gu.rel(out["z"][i], m["z_exact"][i]) for i in range(B)]
    print(name, kw, "t=%.2fs" % dt, "e_z max %.2e" % max(errs), [(s["iters"], s["refines"], s["status"], "%.1e" % s["rel_res"]) for s in out["stats_fwd"]], flush=True)
