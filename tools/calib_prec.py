import os, sys, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from paper_2502_18377_b200 import mpde
for name in sys.argv[1:]:
    B = 4
    bt = synth.make_batch(name, batch=B); g = synth.make_g(name, batch=B); mm = synth.make_mms(name, batch=B); cfg = bt["cfg"]
    ref = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g, opts=mpde.mpde_default_options(tol=1e-11, tol_z=1e-9, max_refine=12, tol_inner=1e-5, precision=3))
    for kw in (dict(precision=0), dict(precision=1), dict(precision=2)):
        o = mpde.mpde_default_options(**kw)
        out = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g, opts=o)
        ez = max(gu.rel(out["z"][i], ref["z"][i]) for i in range(B))
        eg = max(max(gu.rel(out[k][i], ref[k][i]) for i in range(B)) for k in ("grad_c", "grad_b", "grad_omega"))
        om = gu.gpu_solve(cfg.shape, cfg.h, mm["c"], mm["b"], mm["omega"], opts=o)
        em = max(gu.rel(om["z"][i], mm["z_exact"][i]) for i in range(B))
        print(name, kw, f"real e_z {ez:.1e} e_g {eg:.1e} its f/b {np.mean([s['iters'] for s in out['stats_fwd']]):.0f}/{np.mean([s['iters'] for s in out['stats_bwd']]):.0f} st {set(s['status'] for s in out['stats_fwd']+out['stats_bwd'])} | mms e_z {em:.1e}", flush=True)
