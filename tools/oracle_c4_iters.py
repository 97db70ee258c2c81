"""Full oracle fwd + bwd solve of C4 PDE 0 (Jacobi-CG to the oracle's 1e-12 stop); records
the iteration counts used by bench.py's cpu_baseline extrapolation.  Calls only oracle/ and
synth/.  Writes profiles/oracle_c4_iters.json.  (~10 min on one core.)"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from oracle import Problem, assemble
from oracle.neurlp import solve_normal
cfg = synth.CONFIGS["C4"]
bt = synth.make_batch("C4", batch=1)
g = synth.make_g("C4", batch=1)
pr = Problem(cfg.shape, cfg.h)
t0 = time.perf_counter()
A, d, _ = assemble(pr, bt["c"][0], bt["b"][0], bt["omega"][0])
ta = time.perf_counter() - t0
out = {"config": "C4 PDE 0", "assembly_s": ta}
for name, rhs in (("fwd", A.T @ d), ("bwd", g[0].reshape(-1).astype(np.float64))):
    info = {}
    t1 = time.perf_counter()
    solve_normal(A, rhs, method="cg", tol=1e-12, maxiter=100000, info=info, strict=False)
    out[name] = {"iters": info["iters"], "rel_res": info["rel_res"], "seconds": time.perf_counter() - t1}
    print(name, out[name], flush=True)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "profiles", "oracle_c4_iters.json"), "w"), indent=1)
