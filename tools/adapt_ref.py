"""Stop-rule accuracy on real workload data (dev tool, GPU): z from the default options against
a reference solved far past the stop (tol_z 1e-9, up to 8 refinement passes: each fp64 pass
contracts the error by ~tol_inner2, so the reference is accurate to ~1e-9), per PDE the
estimate vs the true relative error, forward and backward.

usage: python tools/adapt_ref.py CONFIG B [option=value ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2502_18377_b200 import mpde  # noqa: E402

name, B = sys.argv[1], int(sys.argv[2])
cfg = synth.CONFIGS[name]
bt = synth.make_batch(name, batch=B)
g = synth.make_g(name, batch=B)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def run(opts):
    s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]), opts=opts)
    z = s.forward(dev(bt["b"]), dev(bt["omega"]))
    torch.cuda.synchronize()
    sf = s.stats_list()
    gc, gb, gw, dz = s.backward(dev(bt["b"]), z, dev(g), want_dz=True)
    torch.cuda.synchronize()
    sb = s.stats_list()
    s.close()
    return z.cpu().numpy().astype(np.float64), dz.cpu().numpy().astype(np.float64), gc.cpu().numpy(), sf, sb


kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = float(v) if "." in v or "e" in v else int(v)
z, dz, gc, sf, sb = run(mpde.mpde_default_options(**kw))
zr, dzr, gcr, sfr, sbr = run(mpde.mpde_default_options(tol_z=1e-9, max_refine=8, max_iters=2000))
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
ez = [rel(z[i], zr[i]) for i in range(B)]
ed = [rel(dz[i], dzr[i]) for i in range(B)]
eg = [rel(gc[i], gcr[i]) for i in range(B)]
print(f"{name} B={B} opts={kw}: fwd iters mean "
      f"{np.mean([x['iters'] for x in sf]):.1f} passes {sorted(set(x['refines'] for x in sf))}; bwd iters mean "
      f"{np.mean([x['iters'] for x in sb]):.1f} passes {sorted(set(x['refines'] for x in sb))}")
print(f"  max e_z {max(ez):.2e} (est max {max(x['err_est'] for x in sf):.2e}, max e_z/est "
      f"{max(e / max(x['err_est'], 1e-30) for e, x in zip(ez, sf)):.2f}); max e_dz {max(ed):.2e} (est max "
      f"{max(x['err_est'] for x in sb):.2e}); max e_grad_c {max(eg):.2e}; reference passes "
      f"{sorted(set(x['refines'] for x in sfr))}/{sorted(set(x['refines'] for x in sbr))}")
w = int(np.argmax(eg))
print(f"  worst grad_c PDE {w}: e_grad_c {eg[w]:.2e}, e_z {ez[w]:.2e}, e_dz {ed[w]:.2e}, fwd passes "
      f"{sf[w]['refines']} est {sf[w]['err_est']:.1e}")
print("  fwd (iters, passes, est, e_z):", [(x["iters"], x["refines"], f"{x['err_est']:.1e}", f"{e:.1e}")
                                          for x, e in zip(sf, ez)])
