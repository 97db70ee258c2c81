"""Write the oracle reference files for the C3 / C4 GPU parity tests (tests/golden/).

Calls only oracle/ and synth/ (the CUDA path is never imported).  For each (config, PDE index)
it assembles A (Eqs. 3-8), solves the forward normal equations (Eq. 9) and the backward
system A^T A d_z = g (Eq. 11) with the oracle's t-slab block-Jacobi PCG (method 'slab', pinned
against SVD / SuperLU / Jacobi-CG by tests/test_oracle_pins.py::test_solver_crosscheck) to a
true normal residual <= 1e-10, and stores z*, d_z and the field gradients of P:240 as float32
(np.savez_compressed) with the residuals, iteration counts and wall times in a JSON sidecar.
g is synth.make_g (N(0,1), seed 77), the parity loss direction 1 of SURVEY §8(c).

  python tools/make_golden.py C4:0 C4:31 C3:0 C3:1      (one process per item, in parallel)
"""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden")
SLAB = {"C3": 4, "C4": 2}


def one(item):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    import synth
    from oracle import Problem, solve_backward, solve_forward
    name, idx = item.split(":")
    idx = int(idx)
    cfg = synth.CONFIGS[name]
    bt = synth.make_batch(name, 1, start=idx)
    g = synth.make_g(name, 1, start=idx)[0].reshape(-1).astype(np.float64)
    pr = Problem(cfg.shape, cfg.h)
    t0 = time.perf_counter()
    from oracle import neurlp
    logf = open(os.path.join(OUT, f"{name.lower()}_pde{idx}.log"), "w")
    orig = neurlp.solve_normal

    def logged(*a, **kw):  # progress lines + no strict raise: the residual reached is recorded
        kw["log"] = lambda it, rel: (logf.write(f"{it} {rel:.3e}\n"), logf.flush())
        kw["strict"] = False
        kw["maxiter"] = 3000
        return orig(*a, **kw)

    neurlp.solve_normal = logged
    f = solve_forward(pr, bt["c"][0], bt["b"][0], bt["omega"][0], method="slab", slab=SLAB[name])
    t1 = time.perf_counter()
    logf.write("bwd\n")
    bw = solve_backward(pr, f, g, method="slab", slab=SLAB[name])
    neurlp.solve_normal = orig
    t2 = time.perf_counter()
    f32 = lambda a: np.asarray(a, dtype=np.float32)
    base = os.path.join(OUT, f"{name.lower()}_pde{idx}")
    np.savez_compressed(base + ".npz", z=f32(f["z"]), dz=f32(bw["dz"]), grad_c=f32(bw["grad_c"]),
                        grad_b=f32(bw["grad_b"]), grad_omega=f32(bw["grad_omega"]))
    fi, bi = f["info"]["solve"], bw["info"]
    meta = {"config": name, "pde_index": idx, "shape": list(cfg.shape), "h": list(cfg.h),
            "method": f"slab (t-slab block-Jacobi PCG, {SLAB[name]} planes per block, SuperLU)",
            "g": "synth.make_g(seed 77)", "fwd": {"iters": fi["iters"], "rel_res": fi["rel_res"],
                                                 "seconds": t1 - t0},
            "bwd": {"iters": bi["iters"], "rel_res": bi["rel_res"], "seconds": t2 - t1},
            "norms": {k: float(np.linalg.norm(v)) for k, v in (("z", f["z"]), ("dz", bw["dz"]),
                                                                ("grad_c", bw["grad_c"]))},
            "writer": "tools/make_golden.py (oracle/ + synth/ only)"}
    json.dump(meta, open(base + ".json", "w"), indent=1)
    return meta


if __name__ == "__main__":
    items = sys.argv[1:] or ["C4:0", "C4:31", "C3:0", "C3:1"]
    os.makedirs(OUT, exist_ok=True)
    with ProcessPoolExecutor(len(items)) as ex:
        for m in ex.map(one, items):
            print(json.dumps(m), flush=True)
