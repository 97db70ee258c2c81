import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu
from test_gpu_parity import _rand_problem
from paper_2502_18377_b200 import mpde
for shape, h, B in (((20, 26), (0.05, 0.04), 3), ((16, 16), (1/15, 1/15), 2)):
    c, b, om, g = _rand_problem(shape, B, 31)
    for kw in ({"precision": 0}, {}, {"precision": 2}, {"levels_max": 1}, {"max_refine": 8}):
        out = gu.gpu_solve(shape, h, c, b, om, g, weights=(1.25, 2.0, 0.75, 0.875), opts=mpde.mpde_default_options(**kw))
        print(shape, kw, [(s["iters"], s["refines"], s["status"], "%.1e" % s["rel_res"]) for s in out["stats_fwd"]], [(s["iters"], s["refines"], s["status"], "%.1e" % s["rel_res"]) for s in out["stats_bwd"]], flush=True)
