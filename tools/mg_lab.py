"""Two-grid lab (dev tool, GPU): dense condensed operator S of one NS (C4-generator) PDE on a
small grid, probed through mpde_apply_schur, and the condition number of S preconditioned by
candidate smoother / coarse-grid combinations (fp64 dense linear algebra).
PCG iterations to 1e-6 ~ 7.3 sqrt(kappa)."""
import os, sys, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from synth import gen
from paper_2502_18377_b200 import mpde

shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,16,16").split(","))
hh = (0.01, 1 / 64, 1 / 64)
D = len(shape)
P = int(np.prod(shape))
NB = 512
gen.CONFIGS["X"] = gen.Config("X", 4, shape, hh, (0.0,) * 3, 1, "ns2d")
bt = synth.make_batch("X", batch=1)
c = gu.to_dev(np.repeat(bt["c"], NB, axis=0))
s = mpde.Solver(shape, hh, c, opts=mpde.mpde_default_options(precision=0))
L = mpde.mpde_hierarchy_query(s.h_, 0, 0, None)[3]
print("levels", [mpde.mpde_hierarchy_query(s.h_, l, 0, None)[:3] for l in range(L)])
dev = "cuda"


def dense(level, Pl):
    cols = []
    for j0 in range(0, Pl, NB):
        x = torch.zeros((NB, Pl), device=dev)
        for k in range(NB):
            if j0 + k < Pl:
                x[k, j0 + k] = 1.0
        y = torch.empty_like(x)
        mpde.mpde_apply_schur(s.h_, level, x, y)
        cols.append(y[: min(NB, Pl - j0)].double())
    torch.cuda.synchronize()
    M = torch.cat(cols, 0).T  # column j = S e_j
    asym = (M - M.T).abs().max().item() / M.abs().max().item()
    return 0.5 * (M + M.T), asym


def precond_dense():
    cols = []
    for j0 in range(0, P, NB):
        x = torch.zeros((NB, P), device=dev)
        for k in range(NB):
            x[k, j0 + k] = 1.0
        z = torch.empty_like(x)
        mpde.mpde_apply_precond(s.h_, x, z)
        cols.append(z.double())
    torch.cuda.synchronize()
    M = torch.cat(cols, 0).T
    return 0.5 * (M + M.T)


S0, a0 = dense(0, P)
shp1 = mpde.mpde_hierarchy_query(s.h_, 1, 0, None)[:D]
P1 = int(np.prod(shp1))
S1, a1 = dense(1, P1)
print("asym", a0, a1)


def prolong_1d(nf, nc):
    Pm = np.zeros((nf, nc))
    for i in range(nf):
        if nf == nc:
            Pm[i, i] = 1
        elif nf % 2 == 0:
            I = i >> 1
            J = I + 1 if i & 1 else I - 1
            J = min(max(J, 0), nc - 1)
            Pm[i, I] += 0.75
            Pm[i, J] += 0.25
        elif i % 2 == 0:
            Pm[i, i >> 1] = 1
        else:
            Pm[i, i >> 1] = 0.5
            Pm[i, (i >> 1) + 1] = 0.5
    return Pm


def kron_all(ms):
    out = ms[0]
    for m in ms[1:]:
        out = np.kron(out, m)
    return out


Pr = torch.tensor(kron_all([prolong_1d(shape[d], shp1[d]) for d in range(D)]), device=dev)
ratio = float(np.prod([shape[d] / shp1[d] for d in range(D)]))  # points per coarse point
R = Pr.T / Pr.T.sum(1, keepdim=True)


def kappa(Bm):
    """condition number of Bm S0 (Bm SPD)."""
    Lc = torch.linalg.cholesky(Bm)
    ev = torch.linalg.eigvalsh(Lc.T @ S0 @ Lc)
    return (ev[-1] / ev[0]).item(), ev[0].item(), ev[-1].item()


def lmax_of(Ms):
    Lc = torch.linalg.cholesky(Ms)
    return torch.linalg.eigvalsh(Lc.T @ S0 @ Lc)[-1].item()


I = torch.eye(P, dtype=torch.float64, device=dev)


def cheb_poly(Minv, nu, ratio_c=60.0):
    """Chebyshev smoother as an operator: e = Q r, Q = p(Minv S) Minv (hi 1.1 lmax, lo lmax/ratio)."""
    lm = lmax_of(Minv)
    hi, lo = 1.1 * lm, lm / ratio_c
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    A = Minv @ S0
    # standard Chebyshev iteration from zero on A x = Minv r
    d = Minv / theta
    x = d.clone()
    for k in range(1, nu):
        rho_new = 1.0 / (2 * sigma - rho)
        d = rho_new * rho * d + (2 * rho_new / delta) * (Minv - A @ x)
        x = x + d
        rho = rho_new
    return x  # x = Q (operator on r)


def two_grid(Q, Sc):
    """symmetric two-grid preconditioner with pre/post smoother Q (pre) and Q^T (post)."""
    Ec = Pr @ torch.linalg.solve(Sc, R)
    Es = I - Q @ S0
    # B = I - (I - Q^T S)(I - Ec S)(I - Q S) S^{-1}  written without S^{-1}
    Bm = Q + Q.T - Q.T @ S0 @ Q  # smoother part
    M1 = (I - Q.T @ S0)
    Bm = Bm + M1 @ Ec @ M1.T
    return 0.5 * (Bm + Bm.T)


def line_blocks(axis, Sm, shp):
    """block-diagonal of Sm over grid lines along `axis` (inverse, dense)."""
    idx = np.arange(int(np.prod(shp))).reshape(shp)
    Binv = torch.zeros_like(Sm)
    lines = np.moveaxis(idx, axis, -1).reshape(-1, shp[axis])
    for ln in lines:
        t = torch.tensor(ln, device=dev)
        blk = Sm[t][:, t]
        Binv[t.unsqueeze(1), t.unsqueeze(0)] = torch.linalg.inv(blk)
    return Binv


def plane_blocks(axes, Sm, shp):
    idx = np.arange(int(np.prod(shp))).reshape(shp)
    other = [a for a in range(D) if a not in axes][0]
    Binv = torch.zeros_like(Sm)
    for k in range(shp[other]):
        t = torch.tensor(np.take(idx, k, axis=other).ravel(), device=dev)
        Binv[t.unsqueeze(1), t.unsqueeze(0)] = torch.linalg.inv(Sm[t][:, t])
    return Binv


Dinv = torch.diag(1.0 / torch.diag(S0))
Mlib = precond_dense()
Lc = torch.linalg.cholesky(Mlib)
ev = torch.linalg.eigvalsh(Lc.T @ S0 @ Lc)
print("library V-cycle: kappa %.3g" % (ev[-1] / ev[0]).item(), "eig counts <0.02,<0.05,<0.1,<0.2,<0.5:",
      [int((ev < t).sum()) for t in (0.02, 0.05, 0.1, 0.2, 0.5)], "lowest", ev[:8].tolist(), flush=True)
G = Pr.T @ S0 @ Pr / ratio
def bmask(shp):
    m = np.zeros(shp, bool)
    for d in range(len(shp)):
        sl = [slice(None)] * len(shp); sl[d] = 0; m[tuple(sl)] = True; sl[d] = -1; m[tuple(sl)] = True
    return torch.tensor(m.ravel(), device=dev, dtype=torch.float64)
wb2 = 1.0
B1 = torch.diag(bmask(shp1))
Q2 = cheb_poly(Dinv, 2)
M1 = (I - Q2.T @ S0)
def tg_kappa(Pm, Sc):
    Ec = Pm @ torch.linalg.solve(Sc, Pm.T)
    Bm = Q2 + Q2.T - Q2.T @ S0 @ Q2 + M1 @ Ec @ M1.T
    return kappa(0.5 * (Bm + Bm.T))[0]
for sc in (1.0, 2.0):
    S1s = S1 + (sc - 1.0) * wb2 * B1
    Lg = torch.linalg.cholesky(G)
    Li = torch.linalg.inv(Lg)
    gev = torch.linalg.eigvalsh(Li @ S1s @ Li.T)
    print(f"bnd scale {sc}: gen-eig(S1s, PtSP/8) range [{gev[0].item():.3g}, {gev[-1].item():.3g}]"
          f"  two-grid kappa {tg_kappa(Pr / ratio ** 0.5, S1s / 1.0 * 1.0) if False else 0:.3g}", flush=True)
    Ec = Pr @ torch.linalg.solve(S1s * ratio, Pr.T)
    Bm = Q2 + Q2.T - Q2.T @ S0 @ Q2 + M1 @ Ec @ M1.T
    print("   two-grid(redisc, scaled) kappa %.3g" % kappa(0.5 * (Bm + Bm.T))[0], flush=True)
print("two-grid Galerkin full coarsening kappa %.3g" % tg_kappa(Pr, Pr.T @ S0 @ Pr), flush=True)
for name, axes in (("t-only", (0,)), ("xy-only", (1, 2)), ("x-only", (1,)), ("tx", (0, 1))):
    Pm = torch.tensor(kron_all([prolong_1d(shape[d], shape[d] // 2 if d in axes else shape[d]) for d in range(D)]), device=dev)
    print(f"two-grid Galerkin semi-coarsening {name}: kappa %.3g" % tg_kappa(Pm, Pm.T @ S0 @ Pm), flush=True)
lm = lmax_of(Dinv)
Ps = (I - (4.0 / 3.0 / lm) * Dinv @ S0) @ Pr
print("two-grid Galerkin smoothed prolongation: kappa %.3g" % tg_kappa(Ps, Ps.T @ S0 @ Ps), flush=True)
