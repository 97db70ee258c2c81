"""Refinement stop margin against converged oracle references (Q14): for C4 (batch 32)
and C3 (16 solves) at several tol_z, the measured errors of the golden PDEs (tests/golden,
written by tools/make_golden.py from oracle/ only) -- e_z and the relative errors of d_z and
the gradients -- and the iteration counts (mean / max over the batch).  GPU tool (gpurun)."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth
from paper_2502_18377_b200 import mpde

GOLD = os.path.join(ROOT, "tests", "golden")
rel = lambda a, b: float(np.linalg.norm(np.asarray(a, np.float64).ravel() - np.asarray(b, np.float64).ravel())
                         / np.linalg.norm(np.asarray(b, np.float64).ravel()))
for name, idxs in (("C4", (0, 31)), ("C3", (0, 1))):
    refs = {}
    for i in idxs:
        f = os.path.join(GOLD, f"{name.lower()}_pde{i}.npz")
        if os.path.exists(f):
            refs[i] = np.load(f)
    if not refs:
        continue
    cfg = synth.CONFIGS[name]
    bt = synth.make_batch(name)
    g = synth.make_g(name)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    for tz in (1e-4, 3e-5, 1e-5):
        s = mpde.Solver(cfg.shape, cfg.h, dev(bt["c"]), opts=mpde.mpde_default_options(tol_z=tz))
        z = s.forward(dev(bt["b"]), dev(bt["omega"]))
        torch.cuda.synchronize()
        sf = s.stats_list()
        gc, gb, gw, dz = s.backward(dev(bt["b"]), z, dev(g), want_dz=True)
        torch.cuda.synchronize()
        sb = s.stats_list()
        s.close()
        row = {"cfg": name, "tol_z": tz,
               "fwd_iters_mean": float(np.mean([x["iters"] for x in sf])), "fwd_iters_max": max(x["iters"] for x in sf),
               "bwd_iters_mean": float(np.mean([x["iters"] for x in sb])), "bwd_iters_max": max(x["iters"] for x in sb),
               "fwd_refines_max": max(x["refines"] for x in sf), "bwd_refines_max": max(x["refines"] for x in sb)}
        for i, r in refs.items():
            row[f"pde{i}"] = {"e_z": rel(z[i].cpu().numpy(), r["z"]), "e_dz": rel(dz[i].cpu().numpy(), r["dz"]),
                              "e_grad_c": rel(gc[i].cpu().numpy(), r["grad_c"]),
                              "e_grad_b": rel(gb[i].cpu().numpy(), r["grad_b"]),
                              "e_grad_omega": rel(gw[i].cpu().numpy(), r["grad_omega"]),
                              "err_est_fwd": sf[i]["err_est"], "err_est_bwd": sb[i]["err_est"]}
        print(json.dumps(row), flush=True)
