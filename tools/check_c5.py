"""C5-shaped (64,128,128) solves: MMS z error and iterations (batch 4), dev tool (GPU)."""
import os, sys, time, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from paper_2502_18377_b200 import mpde
B = 4
mm = synth.make_mms("C5", batch=B)
cfg = synth.CONFIGS["C5"]
t0 = time.time()
out = gu.gpu_solve(cfg.shape, cfg.h, mm["c"], mm["b"], mm["omega"])
em = max(gu.rel(out["z"][i], mm["z_exact"][i]) for i in range(B))
print("C5 mms e_z %.2e" % em, [(s["iters"], s["refines"], s["status"]) for s in out["stats_fwd"]],
      "%.1fs" % (time.time() - t0), flush=True)
bt = synth.make_batch("C5", batch=B)
g = synth.make_g("C5", batch=B)
out = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g)
print("C5 real", [(s["iters"], s["refines"], s["status"]) for s in out["stats_fwd"]],
      [(s["iters"], s["refines"], s["status"]) for s in out["stats_bwd"]], flush=True)
