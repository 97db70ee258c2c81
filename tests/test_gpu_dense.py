"""§8(f) N3: the dense path for tiny problems ("1D ... solved densely").  With
levels_max = 1 and P <= 1024 the whole condensed operator S is probed on the GPU,
inverted exactly (fp64 Gauss-Jordan) and applied as one GEMV per PCG iteration, so each
refinement pass converges in a handful of iterations.  Parity against the oracle's dense
SVD least-squares solve (O5 "tiny")."""
import numpy as np
import pytest

import synth
from oracle import Problem, solve_backward, solve_forward

pytestmark = pytest.mark.gpu

E_Z, E_G = 1e-4, 1e-3


def _dense_opts():
    from paper_2502_18377_b200 import mpde
    return mpde.mpde_default_options(levels_max=1)


def _rand(shape, B, seed):
    rng = np.random.default_rng(seed)
    M, P = 1 + 2 * len(shape), int(np.prod(shape))
    c = rng.normal(0.0, 0.3, (B, M, P))
    c[:, 1] += 1.0  # c_dt = 1 + noise: full column rank (pin P4 / Q19)
    f32 = lambda a: a.astype(np.float32)
    return f32(c), f32(rng.normal(size=(B, P))), f32(rng.normal(size=(B, P))), \
        f32(rng.normal(size=(B, M, P)))


@pytest.mark.parametrize("shape,h", [((16, 16), (1 / 15, 1 / 15)), ((12, 20), (0.05, 0.1)),
                                     ((32, 32), (1 / 31, 1 / 31))])
def test_dense_path_matches_oracle(shape, h):
    import gpu_util as gu
    B = 6
    c, b, om, g = _rand(shape, B, 700 + shape[1])
    out = gu.gpu_solve(shape, h, c, b, om, g, opts=_dense_opts())
    pr = Problem(shape, h)
    # 32x32 has 5120 unknowns: past 'auto''s SVD limit, and its random coefficients are too
    # ill-conditioned for the strict oracle CG -> the oracle's sparse LU
    meth = "lu" if (1 + 2 * len(shape)) * int(np.prod(shape)) > 5000 else "auto"
    for i in range(B):
        f = solve_forward(pr, c[i], b[i], om[i], method=meth)
        bw = solve_backward(pr, f, g[i].reshape(-1).astype(np.float64), method=meth)
        assert gu.rel(out["z"][i], f["z"]) <= E_Z
        assert gu.rel(out["grad_c"][i], bw["grad_c"]) <= E_G
        assert gu.rel(out["grad_b"][i], bw["grad_b"]) <= E_G
        assert gu.rel(out["grad_omega"][i], bw["grad_omega"]) <= E_G
    # exact coarsest solve = the preconditioner is S^-1 (fp32-rounded): a few PCG
    # iterations per refinement pass, no multigrid
    for st in out["stats_fwd"] + out["stats_bwd"]:
        assert st["status"] == "converged", st
        assert st["iters"] <= 6 * max(1, st["refines"]), st


def test_dense_path_c1_batch():
    """C1 heat (BASELINE configs[0]) replicated over a batch of 512 on the dense path: every
    batch element is the same PDE, so every output row equals the oracle's one solve."""
    import gpu_util as gu
    bt = synth.make_batch("C1")
    cfg = bt["cfg"]
    g = synth.make_g("C1")
    B = 512
    rep = lambda a: np.repeat(a, B, axis=0)
    out = gu.gpu_solve(cfg.shape, cfg.h, rep(bt["c"]), rep(bt["b"]), rep(bt["omega"]), rep(g),
                       opts=_dense_opts())
    pr = Problem(cfg.shape, cfg.h)
    f = solve_forward(pr, bt["c"][0], bt["b"][0], bt["omega"][0], method="dense")
    bw = solve_backward(pr, f, g[0].reshape(-1).astype(np.float64), method="dense")
    for i in (0, 1, B // 2, B - 1):
        assert gu.rel(out["z"][i], f["z"]) <= E_Z
        assert gu.rel(out["grad_c"][i], bw["grad_c"]) <= E_G
    # identical inputs -> bit-identical outputs (no batch-position-dependent arithmetic)
    assert np.array_equal(out["z"][0], out["z"][B - 1])
    assert np.array_equal(out["grad_c"][0], out["grad_c"][B - 1])
