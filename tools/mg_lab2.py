"""Semi-coarsening lab (dev tool, GPU): dense S on a small NS grid and rediscretised coarse
operators on t- / xy-coarsened grids (built by the library on restricted c), nested two-grid
preconditioners -> condition numbers.  PCG iterations to 1e-6 ~ 7.3 sqrt(kappa)."""
import os, sys, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import gpu_util as gu, synth
from synth import gen
from paper_2502_18377_b200 import mpde

dev = "cuda"
NB = 512
shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,16,16").split(","))
h0 = (0.01, 1 / 64, 1 / 64)
gen.CONFIGS["X"] = gen.Config("X", 4, shape, h0, (0.0,) * 3, 1, "ns2d")
c0 = synth.make_batch("X", batch=1)["c"][0].astype(np.float64)  # [M][P]


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


def prolong(shf, shc):
    return kron_all([prolong_1d(shf[d], shc[d]) for d in range(len(shf))])


def dense_S(shp, h, c):
    """S of the single PDE with fields c [M][P] on grid shp, h, via the library (level 0)."""
    P = int(np.prod(shp))
    cd = gu.to_dev(np.repeat(c[None].astype(np.float32), NB, axis=0))
    o = mpde.mpde_default_options(precision=0, levels_max=8, coarsest=8)
    s = mpde.Solver(shp, h, cd, opts=o)
    cols = []
    for j0 in range(0, P, NB):
        x = torch.zeros((NB, P), device=dev)
        k = torch.arange(min(NB, P - j0), device=dev)
        x[k, j0 + k] = 1.0
        y = torch.empty_like(x)
        mpde.mpde_apply_schur(s.h_, 0, x, y)
        cols.append(y[: len(k)].double())
    torch.cuda.synchronize()
    s.close()
    M = torch.cat(cols, 0).T
    return 0.5 * (M + M.T)


def coarsen(shf, hf, c, axes):
    shc = tuple((n + 1) // 2 if d in axes else n for d, n in enumerate(shf))
    hc = tuple(hf[d] * ((shf[d] - 1) / (shc[d] - 1)) if d in axes else hf[d] for d in range(len(shf)))
    Pm = prolong(shf, shc)
    R = Pm.T / Pm.T.sum(1, keepdims=True)
    cc = np.stack([R @ c[m] for m in range(c.shape[0])])
    return shc, hc, cc, torch.tensor(Pm, device=dev), float(np.prod(shf) / np.prod(shc))


def cheb(S, nu, ratio_c=60.0):
    """Chebyshev-Jacobi smoother operator Q (e = Q r) on S."""
    Dinv = torch.diag(1.0 / torch.diag(S))
    dsq = torch.diag(torch.diag(S) ** -0.5)
    lm = torch.linalg.eigvalsh(dsq @ S @ dsq)[-1].item()
    hi, lo = 1.1 * lm, lm / ratio_c
    theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sigma = theta / delta
    rho = 1.0 / sigma
    A = Dinv @ S
    d = Dinv / theta
    x = d.clone()
    for _ in range(1, nu):
        rn = 1.0 / (2 * sigma - rho)
        d = rn * rho * d + (2 * rn / delta) * (Dinv - A @ x)
        x = x + d
        rho = rn
    return x


def two_grid(S, Q, Pm, Bc):
    """symmetric two-grid preconditioner of S: smoother Q, prolongation Pm, coarse approx
    inverse Bc (of P^T S P)."""
    n = S.shape[0]
    I = torch.eye(n, dtype=torch.float64, device=dev)
    M1 = I - Q.T @ S
    Bm = Q + Q.T - Q.T @ S @ Q + M1 @ (Pm @ Bc @ Pm.T) @ M1.T
    return 0.5 * (Bm + Bm.T)


def kappa(S, Bm):
    Lc = torch.linalg.cholesky(Bm)
    ev = torch.linalg.eigvalsh(Lc.T @ S @ Lc)
    return (ev[-1] / ev[0]).item()


def report(name, S, Bm):
    try:
        k = kappa(S, Bm)
        print(f"{name:60s} kappa {k:8.3g}  est_its {7.3 * k ** 0.5:5.0f}", flush=True)
    except Exception as e:
        print(name, "not SPD", flush=True)


S0 = dense_S(shape, h0, c0)
Q0 = cheb(S0, 2)
# full coarsening, rediscretised, exact coarse
for axes, tag in (((0, 1, 2), "full"), ((0,), "t"), ((1, 2), "xy")):
    shc, hc, cc, Pm, ratio = coarsen(shape, h0, c0, axes)
    Sc = dense_S(shc, hc, cc)
    report(f"2-grid {tag} redisc {shc}", S0, two_grid(S0, Q0, Pm, torch.linalg.inv(Sc * ratio)))
    report(f"2-grid {tag} galerkin {shc}", S0, two_grid(S0, Q0, Pm, torch.linalg.inv(Pm.T @ S0 @ Pm)))
# nested: t-coarsen, then at level 1 a two-grid with full / xy / t coarsening (rediscretised)
shc, hc, cc, Pm, ratio = coarsen(shape, h0, c0, (0,))
S1 = dense_S(shc, hc, cc)
Q1 = cheb(S1, 2)
for axes2, tag2 in (((0, 1, 2), "full"), ((1, 2), "xy"), ((0,), "t")):
    sh2, h2, c2, P2, r2 = coarsen(shc, hc, cc, axes2)
    if min(sh2) < 6:
        continue
    S2 = dense_S(sh2, h2, c2)
    B1 = two_grid(S1, Q1, P2, torch.linalg.inv(S2 * r2))
    report(f"3-level t -> {tag2} {sh2} (redisc)", S0, two_grid(S0, Q0, Pm, B1 / ratio))
# nu=1 and nu=3 for t-semi
for nu in (1, 3):
    Qn = cheb(S0, nu)
    report(f"2-grid t redisc nu={nu}", S0, two_grid(S0, Qn, Pm, torch.linalg.inv(S1 * ratio)))
