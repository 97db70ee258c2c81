"""GPU parity of the polynomial PDE-expression template: the CUDA
kernels (mpde_template_coeff / mpde_template_grad through the C ABI) against
oracle/template.py on the same seeded inputs, and the full template -> solve -> adjoint ->
dl/dtheta chain against the oracle chain (dense solve)."""
import numpy as np
import pytest
import torch

import synth
from oracle import Problem, solve_backward, solve_forward
from oracle.template import template_coeff, template_grad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gu():
    import gpu_util
    return gpu_util


def _inputs(shape, B, F, G, seed):
    from math import comb
    rng = np.random.default_rng(seed)
    D = len(shape)
    M, P = 1 + 2 * D, int(np.prod(shape))
    K = comb(F + G, G)
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    feat = f32(rng.uniform(-1.5, 1.5, (B, F, P)))
    theta = f32(rng.normal(size=(M + 1, K)))
    gc = f32(rng.normal(size=(B, M, P)))
    gb = f32(rng.normal(size=(B, P)))
    return feat, theta, gc, gb


def _gpu_template(shape, feat, theta, G, gc=None, gb=None, want_feat=True):
    from paper_2502_18377_b200 import mpde
    B, F, P = feat.shape
    M = 1 + 2 * len(shape)
    prob = mpde.make_problem(shape, [0.1] * len(shape), B)
    tm = mpde.make_template(F, G)
    th, fe = torch.from_numpy(theta).cuda(), torch.from_numpy(feat).cuda()
    c = torch.empty((B, M, P), dtype=torch.float32, device="cuda")
    b = torch.empty((B, P), dtype=torch.float32, device="cuda")
    mpde.mpde_template_coeff(prob, tm, th, fe, c, b)
    out = {"c": c.cpu().numpy(), "b": b.cpu().numpy()}
    if gc is not None:
        ws = torch.empty(mpde.mpde_template_workspace_bytes(prob, tm), dtype=torch.uint8,
                         device="cuda")
        gth = torch.empty_like(th)
        gf = torch.empty_like(fe) if want_feat else None
        mpde.mpde_template_grad(prob, tm, th, fe, torch.from_numpy(gc).cuda(),
                                torch.from_numpy(gb).cuda(), gth, gf, ws)
        out["gth"] = gth.cpu().numpy()
        out["gf"] = gf.cpu().numpy() if want_feat else None
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("shape,B,F,G", [((16, 16), 2, 1, 2), ((6, 7, 11), 3, 2, 3),
                                         ((9, 33, 37), 2, 3, 4), ((101, 256), 1, 1, 4),
                                         ((8, 9), 1, 2, 0)])
def test_template_coeff_matches_oracle(shape, B, F, G, gu):
    feat, theta, _, _ = _inputs(shape, B, F, G, 100 + F * 10 + G)
    out = _gpu_template(shape, feat, theta, G)
    for i in range(B):
        c, b = template_coeff(theta, feat[i], G)
        scale = max(np.abs(c).max(), np.abs(b).max())
        assert np.abs(out["c"][i] - c).max() <= 2e-6 * scale
        assert np.abs(out["b"][i] - b).max() <= 2e-6 * scale


@pytest.mark.parametrize("shape,B,F,G", [((16, 16), 2, 1, 2), ((6, 7, 11), 3, 2, 3),
                                         ((9, 33, 37), 2, 3, 4), ((101, 256), 3, 1, 4),
                                         ((8, 9), 1, 2, 0)])
def test_template_grad_matches_oracle(shape, B, F, G, gu):
    """grad_theta (batch-summed, several 1024-point CTAs + a ragged tail) and grad_feat."""
    feat, theta, gc, gb = _inputs(shape, B, F, G, 200 + F * 10 + G)
    out = _gpu_template(shape, feat, theta, G, gc, gb)
    gth, gf = template_grad(theta, feat, G, gc, gb)
    assert gu.rel(out["gth"], gth) <= 1e-5
    assert gu.rel(out["gf"], gf) <= 1e-5
    # deterministic: fixed-order reduction
    out2 = _gpu_template(shape, feat, theta, G, gc, gb, want_feat=False)
    assert np.array_equal(out["gth"], out2["gth"])


def test_template_c4_twin_full_size(gu):
    """C4 at full size (32x64x64, the bench's PDEs): the NS template (degree 1 in
    (U1, U2)) reproduces the generator's coefficient fields, and grad_theta of seeded
    gradients matches the oracle's chain rule."""
    tb = synth.make_template_batch("C4", 4)
    out = _gpu_template((32, 64, 64), tb["feat"], tb["theta"], 1)
    np.testing.assert_array_equal(out["c"], tb["c"])
    np.testing.assert_array_equal(out["b"], 0.0)
    rng = np.random.default_rng(9)
    gc = rng.normal(size=tb["c"].shape).astype(np.float32)
    gb = rng.normal(size=(4, tb["c"].shape[2])).astype(np.float32)
    out = _gpu_template((32, 64, 64), tb["feat"], tb["theta"], 1, gc, gb)
    gth, gf = template_grad(tb["theta"], tb["feat"], 1, gc, gb)
    assert gu.rel(out["gth"], gth) <= 1e-5
    assert gu.rel(out["gf"], gf) <= 1e-5


@pytest.mark.parametrize("shape,h,F,G", [((16, 16), (1 / 15, 1 / 15), 1, 2),
                                         ((10, 12), (0.1, 0.08), 2, 2)])
def test_template_solve_chain_matches_oracle(shape, h, F, G, gu):
    """Template -> forward solve -> adjoint solve -> dl/dtheta, l = <g, z*>, on the GPU
    (all through the C ABI) against the oracle chain (dense SVD solve, chain rule)."""
    from paper_2502_18377_b200 import mpde
    rng = np.random.default_rng(31 + F)
    B = 2
    D = len(shape)
    M, P = 1 + 2 * D, int(np.prod(shape))
    feat, theta, _, _ = _inputs(shape, B, F, G, 300 + F)
    theta *= 0.3
    theta[1, 0] = 1.0  # c_t = 1 (full rank)
    theta = theta.astype(np.float32)
    om = rng.normal(size=(B, P)).astype(np.float32)
    g = rng.normal(size=(B, M, P)).astype(np.float32)

    tm = mpde.make_template(F, G)
    prob = mpde.make_problem(shape, h, B)
    th, fe = gu.to_dev(theta), gu.to_dev(feat)
    c = torch.empty((B, M, P), dtype=torch.float32, device="cuda")
    b = torch.empty((B, P), dtype=torch.float32, device="cuda")
    mpde.mpde_template_coeff(prob, tm, th, fe, c, b)
    s = mpde.Solver(shape, h, c)
    z = s.forward(b, gu.to_dev(om))
    gc, gb, gw, _ = s.backward(b, z, gu.to_dev(g))
    ws = torch.empty(mpde.mpde_template_workspace_bytes(prob, tm), dtype=torch.uint8, device="cuda")
    gth = torch.empty_like(th)
    gf = torch.empty_like(fe)
    mpde.mpde_template_grad(prob, tm, th, fe, gc, gb, gth, gf, ws)
    torch.cuda.synchronize()
    s.close()

    pr = Problem(shape, h)
    gcs, gbs, zs = [], [], []
    for i in range(B):
        # the oracle consumes the same fp32 template output it would receive (O1)
        ci, bi = template_coeff(theta, feat[i], G)
        ci, bi = ci.astype(np.float32), bi.astype(np.float32)
        f = solve_forward(pr, ci, bi, om[i], method="dense")
        bw = solve_backward(pr, f, g[i].reshape(-1).astype(np.float64), method="dense")
        zs.append(f["z"])
        gcs.append(bw["grad_c"])
        gbs.append(bw["grad_b"])
    gth_o, gf_o = template_grad(theta, feat, G, np.array(gcs), np.array(gbs))
    assert gu.rel(z.cpu().numpy().reshape(B, -1), np.array(zs).reshape(B, -1)) <= 1e-4
    assert gu.rel(gth.cpu().numpy(), gth_o) <= 1e-3
    assert gu.rel(gf.cpu().numpy(), gf_o) <= 1e-3
