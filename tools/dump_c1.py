import sys, os, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2502_18377_b200 import mpde
bt = synth.make_batch("C1"); cfg = bt["cfg"]
s = mpde.Solver(cfg.shape, cfg.h, torch.from_numpy(bt["c"]).cuda())
P = s.P
Minv = np.zeros((P, P))
for j in range(P):
    r = torch.zeros((1, P), device="cuda"); r[0, j] = 1
    z = torch.empty_like(r)
    mpde.mpde_apply_precond(s.h_, r, z)
    Minv[:, j] = z[0].cpu().numpy()
out = {"Minv": Minv}
for l in range(2):
    shp = mpde.mpde_hierarchy_query(s.h_, l, 0, None)
    Pl = shp[0] * shp[1]
    d = torch.empty((1, Pl), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 1, d); out[f"dinv{l}"] = d.cpu().numpy()
    lm = torch.empty((1,), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 2, lm); out[f"lmax{l}"] = lm.cpu().numpy()
    cc = torch.empty((1, 5, Pl), device="cuda"); mpde.mpde_hierarchy_query(s.h_, l, 3, cc); out[f"c{l}"] = cc.cpu().numpy()
si = torch.empty((1, 64, 64), device="cuda"); mpde.mpde_hierarchy_query(s.h_, 1, 4, si); out["sinv"] = si.cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c1_dump.npz", **out)
print("ok", out["lmax0"], np.abs(Minv - Minv.T).max(), np.linalg.eigvalsh((Minv + Minv.T) / 2)[[0, -1]])
