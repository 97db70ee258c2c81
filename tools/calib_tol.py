"""Accuracy vs stopping settings: real C4/C2 data (vs a tight GPU solve) and the MMS twins
(vs the closed-form z*).  python tools/calib_tol.py C4"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu  # noqa: E402
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
B = 4
settings = [dict(tol_inner2=3e-4), dict(tol_inner2=3e-3), dict(tol_inner2=1e-2),
            dict(tol_inner2=3e-2), dict(tol_inner2=1e-1), dict(tol_inner=1e-3, tol_inner2=1e-2),
            dict(tol_inner=1e-4, tol_inner2=1e-2), dict(tol_inner=1e-4, tol_inner2=3e-2)]
if len(sys.argv) > 2 and sys.argv[2] == "default":
    settings = [dict()]
bt = synth.make_batch(name, batch=B)
g = synth.make_g(name, batch=B)
mm = synth.make_mms(name, batch=B)
cfg = bt["cfg"]
ref = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g,
                   opts=mpde.mpde_default_options(tol=1e-11, max_refine=12, tol_inner=1e-5, tol_inner2=1e-5, tol_z=1e-9))
for kw in settings:
    o = mpde.mpde_default_options(**kw)
    out = gu.gpu_solve(cfg.shape, cfg.h, bt["c"], bt["b"], bt["omega"], g, opts=o)
    ez = max(gu.rel(out["z"][i], ref["z"][i]) for i in range(B))
    eg = max(max(gu.rel(out[k][i], ref[k][i]) for i in range(B)) for k in ("grad_c", "grad_b", "grad_omega"))
    om = gu.gpu_solve(cfg.shape, cfg.h, mm["c"], mm["b"], mm["omega"], opts=o)
    em = max(gu.rel(om["z"][i], mm["z_exact"][i]) for i in range(B))
    nr = np.mean([s["refines"] for s in out["stats_fwd"]])
    fi = np.mean([s["iters"] for s in out["stats_fwd"]])
    bi = np.mean([s["iters"] for s in out["stats_bwd"]])
    mi = np.mean([s["iters"] for s in om["stats_fwd"]])
    print(f"{name} {kw} real e_z {ez:.1e} e_g {eg:.1e} its f/b {fi:.0f}/{bi:.0f} passes {nr:.1f} | mms e_z {em:.1e} its {mi:.0f}",
          flush=True)
