"""Thin ctypes binding of ``include/mpde.h`` (argument marshalling only).

Every step of the solve runs in ``libmpde.so`` (CUDA, sm_100a).  PyTorch supplies device
memory (tensors, the workspace), streams and process groups; there is no CPU fallback:
if the library or a CUDA device is missing, these functions raise.

Functions keep the C names: ``mpde_workspace_bytes``, ``mpde_build_hierarchy``,
``mpde_solve_fwd``, ``mpde_solve_bwd``, ``mpde_destroy_hierarchy``, ``mpde_sizes``,
``mpde_apply_normal``, ``mpde_apply_schur``, ``mpde_hierarchy_query``,
``mpde_fwd_bwd_host``.  ``Solver`` and ``NeuRLPSolve`` are conveniences on top.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPDE_LIB") or os.path.join(_HERE, "libmpde.so")  # MPDE_LIB: A/B builds


class mpde_problem(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("n", C.c_int32 * 4), ("h", C.c_double * 4),
                ("batch", C.c_int32), ("deriv_order", C.c_int32), ("w_eq", C.c_float),
                ("w_bnd", C.c_float), ("w_deriv", C.c_float), ("w_smooth", C.c_float),
                ("bc", (C.c_int32 * 2) * 4)]


BC_CODES = {"D": 0, "N": 1, "-": 2, 0: 0, 1: 1, 2: 2}


class mpde_options(C.Structure):
    _fields_ = [("tol", C.c_float), ("tol_inner", C.c_float), ("max_iters", C.c_int32),
                ("max_refine", C.c_int32), ("smoother", C.c_int32), ("nu", C.c_int32),
                ("coarsest", C.c_int32), ("levels_max", C.c_int32), ("poll_every", C.c_int32),
                ("jacobi_theta", C.c_float), ("cheb_ratio", C.c_float),
                ("lanczos_steps", C.c_int32), ("precision", C.c_int32),
                ("use_graphs", C.c_int32), ("tol_z", C.c_float), ("tol_inner2", C.c_float),
                ("cf_bf16", C.c_int32), ("krylov", C.c_int32), ("restart", C.c_int32),
                ("grad_steps", C.c_int32), ("tol_adapt", C.c_float)]


class mpde_stats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("refines", C.c_int32), ("status", C.c_int32),
                ("rel_res", C.c_float), ("err_est", C.c_float)]


class mpde_template(C.Structure):
    _fields_ = [("n_feat", C.c_int32), ("degree", C.c_int32)]


STATUS = {0: "converged", 1: "maxiter", 2: "nonfinite", 3: "indefinite"}
_lib = None


def lib():
    """Load libmpde.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2502_18377_b200.build`")
        L = C.CDLL(LIB_PATH)
        P, O, S = C.POINTER(mpde_problem), C.POINTER(mpde_options), C.c_void_p
        vp = C.c_void_p
        L.mpde_default_options.restype = mpde_options
        L.mpde_last_error.restype = C.c_char_p
        L.mpde_sizes.argtypes = [P, O, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int32)]
        L.mpde_workspace_bytes.argtypes = [P, O]
        L.mpde_workspace_bytes.restype = C.c_size_t
        L.mpde_build_hierarchy.argtypes = [P, O, vp, vp, C.c_size_t, S, C.POINTER(vp)]
        L.mpde_solve_fwd.argtypes = [vp, vp, vp, vp, vp, S]
        L.mpde_solve_bwd.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, S]
        L.mpde_solve_fwd_bc.argtypes = [vp, vp, vp, vp, vp, vp, vp, S]
        L.mpde_step_gradient.argtypes = [vp, vp, vp, S]
        L.mpde_solve_bwd_bc.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, S]
        L.mpde_destroy_hierarchy.argtypes = [vp]
        L.mpde_apply_normal.argtypes = [P, vp, vp, vp, S]
        L.mpde_apply_schur.argtypes = [vp, C.c_int32, vp, vp, S]
        L.mpde_apply_precond.argtypes = [vp, vp, vp, S]
        L.mpde_hierarchy_query.argtypes = [vp, C.c_int32, C.c_int32, vp, S]
        L.mpde_batch_sum.argtypes = [vp, C.c_int32, C.c_int64, vp, S]
        L.mpde_profile_end.argtypes = [vp, vp, vp]
        L.mpde_launch_count.restype = C.c_uint64
        L.mpde_host_staging_bytes.argtypes = [P]
        L.mpde_host_staging_bytes.restype = C.c_size_t
        L.mpde_fwd_bwd_host.argtypes = [P, O, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                        C.c_size_t, S]
        T = C.POINTER(mpde_template)
        L.mpde_template_terms.argtypes = [T]
        L.mpde_template_terms.restype = C.c_int32
        L.mpde_template_coeff.argtypes = [P, T, vp, vp, vp, vp, S]
        L.mpde_template_workspace_bytes.argtypes = [P, T]
        L.mpde_template_workspace_bytes.restype = C.c_size_t
        L.mpde_template_grad.argtypes = [P, T, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, S]
        _lib = L
    return _lib


EXPORTS = ["mpde_default_options", "mpde_sizes", "mpde_workspace_bytes", "mpde_build_hierarchy",
           "mpde_solve_fwd", "mpde_solve_bwd", "mpde_solve_fwd_bc", "mpde_solve_bwd_bc", "mpde_step_gradient", "mpde_destroy_hierarchy", "mpde_last_error",
           "mpde_apply_normal", "mpde_apply_schur", "mpde_apply_precond", "mpde_hierarchy_query",
           "mpde_host_staging_bytes", "mpde_fwd_bwd_host", "mpde_batch_sum",
           "mpde_profile_begin", "mpde_profile_end", "mpde_launch_count", "mpde_template_terms",
           "mpde_template_coeff", "mpde_template_workspace_bytes", "mpde_template_grad"]
PROF_CLASSES = ["schur_g", "schur_out", "residual64", "condense", "backsub", "transfer",
                "vector", "scalar", "coarse", "build", "epilogue", "schur_out_l0", "schur_g_l0",
                "schur_march_l0", "schur_march"]


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"mpde error {rc}: {lib().mpde_last_error().decode()}")


def make_problem(shape, h, batch, w_eq=1.0, w_bnd=1.0, w_deriv=1.0, w_smooth=1.0, bc=None):
    """bc: per dim (low, high) face types, 'D' Dirichlet / 'N' Neumann / '-' none (or the
    MPDE_BC_* codes); None = every face Dirichlet."""
    pr = mpde_problem()
    pr.ndim = len(shape)
    for d, (n, hh) in enumerate(zip(shape, h)):
        pr.n[d] = int(n)
        pr.h[d] = float(hh)
    pr.batch = int(batch)
    pr.deriv_order = 2
    pr.w_eq, pr.w_bnd, pr.w_deriv, pr.w_smooth = w_eq, w_bnd, w_deriv, w_smooth
    if bc is not None:
        for d, (lo, hi) in enumerate(bc):
            pr.bc[d][0], pr.bc[d][1] = BC_CODES[lo], BC_CODES[hi]
    return pr


def mpde_default_options(**kw) -> mpde_options:
    o = lib().mpde_default_options()
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dev_f32(t, name):
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
    return t


def mpde_sizes(prob, opts=None):
    nv, nc, nl = C.c_int64(), C.c_int64(), C.c_int32()
    _check(lib().mpde_sizes(C.byref(prob), None if opts is None else C.byref(opts), C.byref(nv),
                            C.byref(nc), C.byref(nl)))
    return nv.value, nc.value, nl.value


def mpde_workspace_bytes(prob, opts):
    n = lib().mpde_workspace_bytes(C.byref(prob), C.byref(opts))
    if n == 0:
        raise RuntimeError("invalid problem/options")
    return n


def mpde_build_hierarchy(prob, opts, coeff, workspace, stream=None):
    h = C.c_void_p()
    _dev_f32(coeff, "coeff")
    _check(lib().mpde_build_hierarchy(C.byref(prob), C.byref(opts), _ptr(coeff), _ptr(workspace),
                                      workspace.numel(), _stream(stream), C.byref(h)))
    return h


def mpde_solve_fwd(h, rhs_b, bnd, z, stats=None, stream=None):
    _check(lib().mpde_solve_fwd(h, _ptr(_dev_f32(rhs_b, "rhs_b")), _ptr(_dev_f32(bnd, "bnd")),
                                _ptr(_dev_f32(z, "z")), _ptr(stats), _stream(stream)))


def mpde_solve_bwd(h, rhs_b, z, g_z, grad_coeff, grad_rhs, grad_bnd, dz=None, stats=None,
                   stream=None):
    _check(lib().mpde_solve_bwd(h, _ptr(rhs_b), _ptr(z), _ptr(_dev_f32(g_z, "g_z")),
                                _ptr(grad_coeff), _ptr(grad_rhs), _ptr(grad_bnd), _ptr(dz),
                                _ptr(stats), _stream(stream)))


def mpde_solve_fwd_bc(h, rhs_b, bnd, bnd_n, z, stats=None, stream=None, lambda_opt=None):
    _check(lib().mpde_solve_fwd_bc(h, _ptr(_dev_f32(rhs_b, "rhs_b")), _ptr(_dev_f32(bnd, "bnd")),
                                   None if bnd_n is None else _ptr(_dev_f32(bnd_n, "bnd_n")),
                                   _ptr(_dev_f32(z, "z")),
                                   None if lambda_opt is None else _ptr(_dev_f32(lambda_opt, "lambda_opt")),
                                   _ptr(stats), _stream(stream)))


def mpde_solve_bwd_bc(h, rhs_b, z, g_z, grad_coeff, grad_rhs, grad_bnd, grad_bnd_n, dz=None,
                      stats=None, stream=None):
    _check(lib().mpde_solve_bwd_bc(h, _ptr(rhs_b), _ptr(z), _ptr(_dev_f32(g_z, "g_z")),
                                   _ptr(grad_coeff), _ptr(grad_rhs), _ptr(grad_bnd),
                                   _ptr(grad_bnd_n), _ptr(dz), _ptr(stats), _stream(stream)))


def mpde_step_gradient(h, z, grad_h, stream=None):
    """dl/dh [B][ndim] after mpde_solve_bwd (options.grad_steps = 1)."""
    _check(lib().mpde_step_gradient(h, _ptr(_dev_f32(z, "z")), _ptr(_dev_f32(grad_h, "grad_h")),
                                    _stream(stream)))
    return grad_h


def mpde_destroy_hierarchy(h):
    _check(lib().mpde_destroy_hierarchy(h))


def mpde_apply_normal(prob, coeff, z, q, stream=None):
    _check(lib().mpde_apply_normal(C.byref(prob), _ptr(coeff), _ptr(z), _ptr(q), _stream(stream)))


def mpde_apply_schur(h, level, x, y, stream=None):
    _check(lib().mpde_apply_schur(h, int(level), _ptr(x), _ptr(y), _stream(stream)))


def mpde_apply_precond(h, r, z, stream=None):
    _check(lib().mpde_apply_precond(h, _ptr(r), _ptr(z), _stream(stream)))


def mpde_hierarchy_query(h, level, what, dst, stream=None):
    if what in (0, 5, 6):
        arr = (C.c_int32 * (5 if what == 6 else 4))()
        _check(lib().mpde_hierarchy_query(h, int(level), int(what), C.cast(arr, C.c_void_p),
                                          _stream(stream)))
        return list(arr)
    _check(lib().mpde_hierarchy_query(h, int(level), int(what), _ptr(dst), _stream(stream)))
    return dst


def mpde_batch_sum(x, out, stream=None):
    B = x.shape[0]
    _check(lib().mpde_batch_sum(_ptr(x), B, x.numel() // B, _ptr(out), _stream(stream)))
    return out


def mpde_launch_count():
    return int(lib().mpde_launch_count())


def mpde_profile_begin():
    _check(lib().mpde_profile_begin())


def mpde_profile_end():
    """-> (dict class -> (ms, launches), pts[32])"""
    n = len(PROF_CLASSES)
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    pts = (C.c_uint64 * 32)()
    _check(lib().mpde_profile_end(C.cast(ms, C.c_void_p), C.cast(cnt, C.c_void_p),
                                  C.cast(pts, C.c_void_p)))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(PROF_CLASSES)}, list(pts)


def mpde_host_staging_bytes(prob):
    return lib().mpde_host_staging_bytes(C.byref(prob))


def mpde_fwd_bwd_host(prob, opts, c_h, b_h, om_h, g_h, z_h, gc_h, gb_h, gw_h, staging, workspace,
                      stream=None):
    """All *_h are CPU (ideally pinned) float32 tensors; staging/workspace are CUDA uint8."""
    _check(lib().mpde_fwd_bwd_host(C.byref(prob), C.byref(opts), _ptr(c_h), _ptr(b_h), _ptr(om_h),
                                   _ptr(g_h), _ptr(z_h), _ptr(gc_h), _ptr(gb_h), _ptr(gw_h),
                                   _ptr(staging), _ptr(workspace), workspace.numel(),
                                   _stream(stream)))


def make_template(n_feat, degree):
    t = mpde_template()
    t.n_feat, t.degree = int(n_feat), int(degree)
    return t


def mpde_template_terms(tmpl):
    return int(lib().mpde_template_terms(C.byref(tmpl)))


def mpde_template_coeff(prob, tmpl, theta, feat, coeff, rhs_b, stream=None):
    """theta [|M|+1][K], feat [B][F][P] -> coeff [B][|M|][P], rhs_b [B][P] (all CUDA fp32)."""
    _check(lib().mpde_template_coeff(C.byref(prob), C.byref(tmpl), _ptr(_dev_f32(theta, "theta")),
                                     _ptr(_dev_f32(feat, "feat")), _ptr(_dev_f32(coeff, "coeff")),
                                     _ptr(_dev_f32(rhs_b, "rhs_b")), _stream(stream)))


def mpde_template_workspace_bytes(prob, tmpl):
    n = lib().mpde_template_workspace_bytes(C.byref(prob), C.byref(tmpl))
    if n == 0:
        raise RuntimeError("invalid problem/template")
    return n


def mpde_template_grad(prob, tmpl, theta, feat, grad_coeff, grad_rhs, grad_theta, grad_feat,
                       workspace, stream=None):
    _check(lib().mpde_template_grad(C.byref(prob), C.byref(tmpl), _ptr(theta), _ptr(feat),
                                    _ptr(_dev_f32(grad_coeff, "grad_coeff")),
                                    _ptr(_dev_f32(grad_rhs, "grad_rhs")),
                                    _ptr(_dev_f32(grad_theta, "grad_theta")), _ptr(grad_feat),
                                    _ptr(workspace), workspace.numel(), _stream(stream)))


# ------------------------------------------------------------------------------------
class Solver:
    """Owns a workspace and a hierarchy for one batch of coefficient fields.

    c: [B][M][P] float32 CUDA tensor (kept alive by the Solver).  Forward and backward
    follow mpde.h; stats are returned as a list of dicts after a stream sync.
    """

    def __init__(self, shape, h, c, opts=None, weights=(1.0, 1.0, 1.0, 1.0), stream=None, bc=None):
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required (no CPU fallback)")
        self.shape, self.h = tuple(shape), tuple(h)
        self.B, self.M, self.P = c.shape
        self.prob = make_problem(shape, h, self.B, *weights, bc=bc)
        self.D = len(self.shape)
        self.opts = opts if opts is not None else mpde_default_options()
        self.c = _dev_f32(c, "c")
        nbytes = mpde_workspace_bytes(self.prob, self.opts)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=c.device)
        self.stats = torch.zeros((self.B, 5), dtype=torch.int32, device=c.device)
        self.h_ = mpde_build_hierarchy(self.prob, self.opts, self.c, self.ws, stream)

    def forward(self, b, omega, stream=None, omega_n=None, want_lambda=False):
        """omega_n: [B][D][P] Neumann data (faces of type 'N'); None = 0.  want_lambda: also
        return the duals lambda* [B][2+5D][P] (mpde.h mpde_solve_fwd_bc layout)."""
        z = torch.empty((self.B, self.M, self.P), dtype=torch.float32, device=self.c.device)
        lam = (torch.empty((self.B, 2 + 5 * self.D, self.P), dtype=torch.float32, device=self.c.device)
               if want_lambda else None)
        mpde_solve_fwd_bc(self.h_, b, omega, omega_n, z, self.stats, stream, lambda_opt=lam)
        return (z, lam) if want_lambda else z

    def backward(self, b, z, g, want_dz=False, stream=None, want_grad_omega_n=False):
        """-> (grad_c, grad_b, grad_omega, dz) or, with want_grad_omega_n, the same plus
        dl/domega_n [B][D][P]."""
        gc = torch.empty_like(self.c)
        gb = torch.empty((self.B, self.P), dtype=torch.float32, device=self.c.device)
        gw = torch.empty_like(gb)
        dz = torch.empty_like(self.c) if want_dz else None
        gwn = (torch.empty((self.B, self.D, self.P), dtype=torch.float32, device=self.c.device)
               if want_grad_omega_n else None)
        mpde_solve_bwd_bc(self.h_, b, z, g, gc, gb, gw, gwn, dz, self.stats, stream)
        if want_grad_omega_n:
            return gc, gb, gw, dz, gwn
        return gc, gb, gw, dz

    def step_gradient(self, z, stream=None):
        """dl/dh_d [B][D] for the last backward (needs opts.grad_steps = 1)."""
        gh = torch.empty((self.B, self.D), dtype=torch.float32, device=self.c.device)
        return mpde_step_gradient(self.h_, z, gh, stream)

    def stats_list(self):
        s = self.stats.cpu()
        out = []
        for row in s:
            rel = row[3:4].view(torch.float32).item()
            est = row[4:5].view(torch.float32).item()
            out.append({"iters": int(row[0]), "refines": int(row[1]),
                        "status": STATUS.get(int(row[2]), str(int(row[2]))), "rel_res": rel,
                        "err_est": est})
        return out

    def close(self):
        if self.h_ is not None:
            mpde_destroy_hierarchy(self.h_)
            self.h_ = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NeuRLPSolve(torch.autograd.Function):
    """z* = solve(c, b, omega); backward returns (dl/dc, dl/db, dl/domega) via Eq. 11."""

    @staticmethod
    def forward(ctx, c, b, omega, shape, h, opts):
        s = Solver(shape, h, c.contiguous(), opts)
        z = s.forward(b.contiguous(), omega.contiguous())
        ctx.solver = s
        ctx.save_for_backward(b, z)
        return z

    @staticmethod
    def backward(ctx, gz):
        b, z = ctx.saved_tensors
        gc, gb, gw, _ = ctx.solver.backward(b.contiguous(), z, gz.contiguous())
        ctx.solver.close()
        return gc, gb, gw, None, None, None
