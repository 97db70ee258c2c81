"""§8(f) N1: FGMRES(m) with the same V-cycle (the paper's Krylov method), selected by
mpde_options.krylov = 1.  z* is unique (Q19), so the bar is the same as PCG's: parity with
the fp64 oracle (e_z <= 1e-4, e_g <= 1e-3), and the manufactured solutions at full size."""
import numpy as np
import pytest

import synth
from oracle import Problem, solve_backward, solve_forward

pytestmark = pytest.mark.gpu

E_Z, E_G = 1e-4, 1e-3


def _opts(**kw):
    from paper_2502_18377_b200 import mpde
    return mpde.mpde_default_options(krylov=1, **kw)


def _rand(shape, B, seed):
    rng = np.random.default_rng(seed)
    M, P = 1 + 2 * len(shape), int(np.prod(shape))
    c = rng.normal(0.0, 0.5, (B, M, P))
    c[:, 1] += 1.0
    f32 = lambda a: a.astype(np.float32)
    return f32(c), f32(rng.normal(size=(B, P))), f32(rng.normal(size=(B, P))), \
        f32(rng.normal(size=(B, M, P)))


@pytest.mark.parametrize("shape,h,B,restart", [((16, 16), (1 / 15, 1 / 15), 2, 20),
                                               ((20, 26), (0.05, 0.04), 3, 4),
                                               ((8, 9, 10), (0.1, 0.08, 0.07), 2, 8)])
def test_fgmres_matches_oracle(shape, h, B, restart):
    """Random problems (several tiles + ragged tails); restart 4 / 8 forces restart cycles."""
    import gpu_util as gu
    c, b, om, g = _rand(shape, B, 900 + restart)
    out = gu.gpu_solve(shape, h, c, b, om, g, opts=_opts(restart=restart))
    pr = Problem(shape, h)
    method = "dense" if pr.P * (1 + 2 * len(shape)) <= 5000 else "lu"
    for i in range(B):
        f = solve_forward(pr, c[i], b[i], om[i], method=method)
        bw = solve_backward(pr, f, g[i].reshape(-1).astype(np.float64), method=method)
        assert out["stats_fwd"][i]["status"] == "converged", out["stats_fwd"][i]
        assert out["stats_bwd"][i]["status"] == "converged", out["stats_bwd"][i]
        assert gu.rel(out["z"][i], f["z"]) <= E_Z
        for k in ("grad_c", "grad_b", "grad_omega"):
            assert gu.rel(out[k][i], bw[k]) <= E_G, k


@pytest.mark.parametrize("shape", [(16, 20, 24), (20, 32, 32)])
def test_fgmres_and_pcg_agree(shape):
    """Larger 3D random problems (the (20,32,32) level 0 runs the t-blocked pass-2 kernel):
    z* is unique, so FGMRES and PCG (parity-tested against the oracle) give the same z."""
    import gpu_util as gu
    h = (0.05, 0.05, 0.05)
    c, b, om, _ = _rand(shape, 2, 41)
    zf = gu.gpu_solve(shape, h, c, b, om, opts=_opts())
    zp = gu.gpu_solve(shape, h, c, b, om)
    for i in range(2):
        assert zf["stats_fwd"][i]["status"] == "converged"
        assert gu.rel(zf["z"][i], zp["z"][i]) <= 2 * E_Z


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_fgmres_mms_full_size(name):
    """P2 at full size (C4: the bench workload, full batch of 32): FGMRES recovers the
    closed-form solution, in an iteration count comparable to PCG's."""
    import gpu_util as gu
    m = synth.make_mms(name)
    cfg = m["cfg"]
    out = gu.gpu_solve(cfg.shape, cfg.h, m["c"], m["b"], m["omega"], opts=_opts())
    ref = gu.gpu_solve(cfg.shape, cfg.h, m["c"], m["b"], m["omega"])
    errs = [gu.rel(out["z"][i], m["z_exact"][i]) for i in range(m["c"].shape[0])]
    its = [s["iters"] for s in out["stats_fwd"]]
    its_pcg = [s["iters"] for s in ref["stats_fwd"]]
    print(name, "FGMRES max e_z", max(errs), "iters", min(its), max(its),
          "| PCG iters", min(its_pcg), max(its_pcg))
    assert max(errs) <= E_Z
    assert all(s["status"] == "converged" for s in out["stats_fwd"])
    assert max(its) <= 2 * max(its_pcg) + 20


def test_fgmres_zero_rhs():
    """b = 0, omega = 0 -> z* = 0 exactly, nothing to iterate (GM_BEGIN with ||r0|| = 0)."""
    import gpu_util as gu
    shape, h = (12, 14), (0.1, 0.1)
    c, _, _, g = _rand(shape, 2, 5)
    P = int(np.prod(shape))
    z0 = np.zeros((2, P), np.float32)
    out = gu.gpu_solve(shape, h, c, z0, z0, g, opts=_opts())
    assert np.all(out["z"] == 0.0)
    assert np.all(out["grad_c"] == 0.0)


def test_fgmres_rejects_bad_restart():
    from paper_2502_18377_b200 import mpde
    import torch
    shape, h = (12, 12), (0.1, 0.1)
    c, _, _, _ = _rand(shape, 1, 6)
    with pytest.raises(RuntimeError):
        mpde.Solver(shape, h, torch.from_numpy(c).cuda(), opts=_opts(restart=33))
