"""Refinement stop margin (Q14): iterations and measured errors at several tol_z.

For C2, C3 and C4 (MMS twins: exact z known in closed form) runs fwd + bwd
on the first `n` PDEs at each tol_z and prints mean PCG iterations, the largest e_z against the
exact solution and the largest error estimate the library reported.  GPU tool (gpurun)."""
import json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2502_18377_b200 import mpde

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rows = []
for name in ("C2", "C3", "C4"):
    m = synth.make_mms(name, n)
    cfg = m["cfg"]
    g = synth.make_g(name, n)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    for tz in (1e-4, 3e-5, 1e-5, 3e-6):
        opts = mpde.mpde_default_options(tol_z=tz)
        s = mpde.Solver(cfg.shape, cfg.h, dev(m["c"]), opts=opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        z = s.forward(dev(m["b"]), dev(m["omega"]))
        torch.cuda.synchronize()
        sf = s.stats_list()
        s.backward(dev(m["b"]), z, dev(g))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        sb = s.stats_list()
        s.close()
        zz = z.cpu().numpy().astype(np.float64)
        ez = [np.linalg.norm(zz[i] - m["z_exact"][i]) / np.linalg.norm(m["z_exact"][i]) for i in range(n)]
        r = {"cfg": name, "tol_z": tz, "fwd_iters": float(np.mean([x["iters"] for x in sf])),
             "bwd_iters": float(np.mean([x["iters"] for x in sb])),
             "fwd_refines": float(np.mean([x["refines"] for x in sf])),
             "e_z_max": float(max(ez)), "est_max": float(max(x["err_est"] for x in sf)),
             "ratio_max": float(max(e / max(x["err_est"], 1e-30) for e, x in zip(ez, sf))),
             "seconds": dt}
        rows.append(r)
        print(json.dumps(r), flush=True)
