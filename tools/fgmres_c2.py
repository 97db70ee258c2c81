"""MMS twins: max e_z and iterations for FGMRES at several tol_inner2 (and PCG for reference).
python tools/fgmres_c2.py C2 [C3 C4]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu  # noqa: E402
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

for name in sys.argv[1:]:
    m = synth.make_mms(name)
    cfg = m["cfg"]
    for kw in [{}, {"krylov": 1}, {"krylov": 1, "tol_inner2": 1e-3}, {"krylov": 1, "tol_inner2": 3e-4},
               {"krylov": 1, "tol_z": 3e-5}]:
        out = gu.gpu_solve(cfg.shape, cfg.h, m["c"], m["b"], m["omega"], opts=mpde.mpde_default_options(**kw))
        errs = [gu.rel(out["z"][i], m["z_exact"][i]) for i in range(m["c"].shape[0])]
        its = [s["iters"] for s in out["stats_fwd"]]
        ref = [s["refines"] for s in out["stats_fwd"]]
        est = [s["err_est"] for s in out["stats_fwd"]]
        k = int(np.argmax(errs))
        print(name, kw, f"max e_z {max(errs):.2e} (pde {k}: est {est[k]:.2e}, refines {ref[k]}, its {its[k]}) "
              f"mean its {np.mean(its):.1f} max its {max(its)}", flush=True)
