"""Quick GPU check of the one-kernel t-marching S apply (march.cu) against the two-pass
kernels (MPDE_MARCH=0) on random problems: max relative difference of y = S x, and the event
time of one apply at C4 level-0 size.  Usage: python tools/march_check.py"""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_2502_18377_b200 import mpde
shape = tuple(json.loads(sys.argv[1])); B = int(sys.argv[2]); out = sys.argv[3]
rng = np.random.default_rng(7)
M, P = 7, int(np.prod(shape))
c = rng.normal(0.0, 0.5, (B, M, P)); c[:, 1] += 1.0
h = (0.02, 0.03, 0.025)
s = mpde.Solver(shape, h, torch.from_numpy(c.astype(np.float32)).cuda(), weights=(1.25, 2.0, 0.75, 0.875))
x = torch.from_numpy(rng.normal(size=(B, P)).astype(np.float32)).cuda()
y = torch.empty_like(x)
mpde.mpde_apply_schur(s.h_, 0, x, y); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): mpde.mpde_apply_schur(s.h_, 0, x, y)
e1.record(); torch.cuda.synchronize()
pc = torch.empty_like(x); mpde.mpde_apply_precond(s.h_, x, pc); torch.cuda.synchronize()
np.savez(out, y=y.cpu().numpy(), pc=pc.cpu().numpy(), us=e0.elapsed_time(e1) / 20 * 1e3,
         v=np.array(mpde.mpde_hierarchy_query(s.h_, 0, 5, None)))
"""
res = []
for shape, B in [((7, 16, 64), 2), ((9, 24, 32), 2), ((20, 32, 32), 4), ((11, 40, 64), 2), ((8, 64, 128), 2),
                 ((32, 64, 64), 32)]:
    outs = {}
    for tag, env in (("march", {"MPDE_MARCH": "2"}), ("twopass", {"MPDE_MARCH": "0"})):
        f = f"/tmp/mc_{tag}.npz"
        r = subprocess.run([sys.executable, "-c", CHILD, json.dumps(shape), str(B), f], cwd=ROOT,
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=300)
        if r.returncode:
            print(tag, shape, "FAILED", r.stderr[-2000:], flush=True)
            break
        outs[tag] = dict(np.load(f))
    if len(outs) < 2:
        continue
    a, b = outs["march"], outs["twopass"]
    ey = float(np.abs(a["y"] - b["y"]).max() / np.abs(b["y"]).max())
    ep = float(np.abs(a["pc"] - b["pc"]).max() / np.abs(b["pc"]).max())
    row = {"shape": shape, "B": B, "rel_y": ey, "rel_precond": ep, "us_march": float(a["us"]),
           "us_twopass": float(b["us"]), "variant": a["v"].tolist()}
    print(json.dumps(row), flush=True)
