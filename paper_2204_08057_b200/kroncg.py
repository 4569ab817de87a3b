"""Thin ctypes binding of libkroncg (include/kroncg.h) -- argument marshalling only.

Every step of the solve runs in the library's CUDA kernels; there is no CPU fallback: if the
shared library is missing or cannot be loaded, importing this module raises.  PyTorch is used
only for device memory (workspace, inputs, outputs) and the CUDA stream.

Functions keep the C names: kron_cg_workspace_size, kron_cg_create, kron_cg_solve,
sylvester_solve, kron_cg_solve_host, sylvester_solve_host, kron_cg_apply, kron_cg_rhs,
sylvester_factor, kcg_last_error, kcg_status_string, kron_cg_destroy.  ``KronCG`` wraps a
context around torch tensors.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KCG_LIB_PATH") or os.path.join(_HERE, "lib", "libkroncg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libkroncg.so not built ({LIB_PATH}); run __graft_entry__.build()")
_lib = C.CDLL(LIB_PATH)

# status codes (kcg_status)
KCG_OK, KCG_NOT_CONVERGED, KCG_E_ARG, KCG_E_SHAPE, KCG_E_CONFIG = 0, 1, 2, 3, 4
KCG_E_NONFINITE, KCG_E_BREAKDOWN, KCG_E_CUDA, KCG_E_STATE = 5, 6, 7, 9
KCG_PRIOR_LAPLACIAN, KCG_PRIOR_D2 = 0, 1
KCG_LAYOUT_ROW_MAJOR, KCG_LAYOUT_NESTED = 0, 1
KCG_PRECOND_NONE, KCG_PRECOND_BLOCK_JACOBI = 0, 1
KCG_CG_SINGLE_PASS, KCG_CG_HS = 0, 1


class kcg_desc(C.Structure):
    _fields_ = [("level", C.c_int), ("n_freq", C.c_int), ("n_comp", C.c_int),
                ("n_patches", C.c_int), ("prior", C.c_int), ("layout", C.c_int),
                ("precond", C.c_int), ("host_staging", C.c_int), ("history_cap", C.c_int),
                ("lanczos_cap", C.c_int), ("lanczos_store", C.c_int), ("cg_variant", C.c_int)]


class kcg_report(C.Structure):
    _fields_ = [("status", C.c_int), ("converged", C.c_int), ("iterations", C.c_int),
                ("n_systems", C.c_int), ("iterations_per", C.POINTER(C.c_int)),
                ("rel_residual", C.c_double), ("rel_residual_true", C.c_double),
                ("wall_time_s", C.c_double), ("loop_time_s", C.c_double),
                ("system_iterations", C.c_longlong), ("loop_bytes", C.c_double),
                ("peak_mem_bytes", C.c_size_t), ("history", C.POINTER(C.c_double)),
                ("history_len", C.c_int), ("kernel_launches", C.c_longlong)]


_vp, _dp, _ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
_ctxp = C.c_void_p


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


kron_cg_workspace_size = _sig("kron_cg_workspace_size", C.c_size_t, [C.POINTER(kcg_desc)])
kron_cg_create = _sig("kron_cg_create", C.c_int,
                      [C.POINTER(kcg_desc), _vp, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp,
                       C.POINTER(_ctxp)])
_solve_args = [_ctxp, _vp, _vp, C.c_double, C.c_int, C.POINTER(kcg_report)]
kron_cg_solve = _sig("kron_cg_solve", C.c_int, _solve_args)
sylvester_solve = _sig("sylvester_solve", C.c_int, _solve_args)
kron_cg_solve_host = _sig("kron_cg_solve_host", C.c_int, _solve_args)
sylvester_solve_host = _sig("sylvester_solve_host", C.c_int, _solve_args)
sylvester_lanczos_solve = _sig("sylvester_lanczos_solve", C.c_int, _solve_args)
sylvester_lanczos_solve_host = _sig("sylvester_lanczos_solve_host", C.c_int, _solve_args)
kron_cg_solve_b = _sig("kron_cg_solve_b", C.c_int, _solve_args)
kron_cg_solve_x0 = _sig("kron_cg_solve_x0", C.c_int, [_ctxp, _vp, _vp, _vp, C.c_double, C.c_int, C.POINTER(kcg_report)])
sylvester_kohler_solve = _sig("sylvester_kohler_solve", C.c_int, _solve_args)
posterior_variance = _sig("posterior_variance", C.c_int,
                          [_ctxp, C.c_int, C.c_ulonglong, _vp, _vp, C.c_double, C.c_int, C.POINTER(kcg_report)])
kron_cg_solve_host_many = _sig("kron_cg_solve_host_many", C.c_int,
                               [_ctxp, C.c_int, C.POINTER(_vp), C.POINTER(_vp), C.c_double, C.c_int,
                                C.POINTER(kcg_report)])
kron_cg_apply = _sig("kron_cg_apply", C.c_int, [_ctxp, _vp, _vp])
kron_cg_rhs = _sig("kron_cg_rhs", C.c_int, [_ctxp, _vp, _vp])
sylvester_factor = _sig("sylvester_factor", C.c_int, [_ctxp, _vp, _vp])
kcg_last_error = _sig("kcg_last_error", C.c_char_p, [_ctxp])


class kcg_slab(C.Structure):
    _fields_ = [("nranks", C.c_int), ("rank0", C.c_int), ("nlocal", C.c_int), ("peer_ws", C.c_void_p * 8)]


kron_cg_workspace_size_slab = _sig("kron_cg_workspace_size_slab", C.c_size_t, [C.POINTER(kcg_desc), C.c_int])
kron_cg_create_slab = _sig("kron_cg_create_slab", C.c_int,
                           [C.POINTER(kcg_desc), C.POINTER(kcg_slab), _vp, _vp, _vp, _vp, _vp, C.c_size_t,
                            _vp, C.POINTER(_ctxp)])
kcg_ipc_export = _sig("kcg_ipc_export", C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_size_t)])
kcg_ipc_import = _sig("kcg_ipc_import", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_vp), C.POINTER(_vp)])
kcg_ipc_close = _sig("kcg_ipc_close", C.c_int, [_vp])
kcg_slab_probe_put = _sig("kcg_slab_probe_put", C.c_int, [_ctxp, C.c_double])
kcg_slab_probe_get = _sig("kcg_slab_probe_get", C.c_int, [_ctxp, C.POINTER(C.c_double)])
kcg_status_string = _sig("kcg_status_string", C.c_char_p, [C.c_int])
kron_cg_destroy = _sig("kron_cg_destroy", None, [_ctxp])

EXPORTS = ["kron_cg_workspace_size", "kron_cg_create", "kron_cg_solve", "sylvester_solve",
           "kron_cg_solve_host", "sylvester_solve_host", "kron_cg_apply", "kron_cg_rhs",
           "sylvester_factor", "kcg_last_error", "kcg_status_string", "kron_cg_destroy",
           "kron_cg_workspace_size_slab", "kron_cg_create_slab", "kcg_ipc_export", "kcg_ipc_import",
           "kcg_ipc_close", "kcg_slab_probe_put", "kcg_slab_probe_get", "sylvester_lanczos_solve", "sylvester_lanczos_solve_host",
           "kron_cg_solve_b", "posterior_variance", "sylvester_kohler_solve", "kron_cg_solve_host_many",
           "kron_cg_solve_x0"]


class KcgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{kcg_status_string(status).decode()}: {msg}")
        self.status = status


def _ptr(a) -> int:
    """Raw pointer of a torch tensor (device or host) or numpy array."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class SolveReport(dict):
    """Host-side copy of kcg_report (plus the per-system iterations and history)."""


class KronCG:
    """One library context over ``n_patches`` faces sharing (level, n, k).

    Parameters are host numpy arrays in the C-ABI layouts (A [P][n][k], noise_prec [P][n],
    prior_scale [P][k], kappa2 [P]); hits an optional torch CUDA tensor [P][side][side].
    precond: "none" (the paper's CG) or "block_jacobi" (pixel-block Jacobi, reading R10).
    prior: "laplacian" (Q0 = kappa2 I + L, the configs) or "d2" (Q0 = D^2 + kappa2 I, the paper's).
    layout: "row" (pixel y*side + x) or "nested" (HEALPix NESTED inside the face, reading R1): Y, mu,
    hits and the apply / rhs arguments keep their [..][side][side] shapes, read as flat [N] vectors.
    lanczos_cap: > 0 provisions the block-Lanczos route (``lanczos``, Alg. SylvSolver) for up to that
    many Lanczos steps; lanczos_store keeps the whole basis in HBM (one assembly pass) instead of
    the paper's second Lanczos pass.
    cg_variant: "single_pass" (Chronopoulos-Gear with recomputation, one reduction per iteration)
    or "hs" (textbook Hestenes-Stiefel CG, Alg. CG, two reductions) -- reading R9.
    """

    def __init__(self, level, A, noise_prec, prior_scale, kappa2, hits=None, device=None,
                 host_staging=False, history_cap=0, stream=None, precond="none", layout="row",
                 prior="laplacian", lanczos_cap=0, lanczos_store=False, cg_variant="single_pass"):
        import torch
        A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
        if A.ndim == 2:
            A = A[None]
        P, n, k = A.shape
        self.noise_prec = np.ascontiguousarray(np.asarray(noise_prec, dtype=np.float64).reshape(P, n))
        self.prior_scale = np.ascontiguousarray(np.asarray(prior_scale, dtype=np.float64).reshape(P, k))
        self.kappa2 = np.ascontiguousarray(np.asarray(kappa2, dtype=np.float64).reshape(P))
        self.A = A
        self.level, self.P, self.n, self.k = level, P, n, k
        self.side = 1 << level
        self.N = self.side * self.side
        self.device = torch.device(device if device is not None else "cuda")
        self.shape_Y = (P, n, self.side, self.side)
        self.shape_mu = (P, k, self.side, self.side)
        pc = {"none": KCG_PRECOND_NONE, "block_jacobi": KCG_PRECOND_BLOCK_JACOBI}[precond]
        lay = {"row": KCG_LAYOUT_ROW_MAJOR, "nested": KCG_LAYOUT_NESTED}[layout]
        pr = {"laplacian": KCG_PRIOR_LAPLACIAN, "d2": KCG_PRIOR_D2}[prior]
        cv = {"single_pass": KCG_CG_SINGLE_PASS, "hs": KCG_CG_HS}[cg_variant]
        self.desc = kcg_desc(level, n, k, P, pr, lay,
                             pc, int(host_staging), int(history_cap), int(lanczos_cap),
                             int(bool(lanczos_store)), cv)
        ws = kron_cg_workspace_size(C.byref(self.desc))
        if ws == 0:
            raise KcgError(KCG_E_SHAPE, "invalid descriptor")
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        self.hits = None
        if hits is not None:
            self.hits = hits.to(device=self.device, dtype=torch.float64).contiguous()
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        ctx = _ctxp()
        st = kron_cg_create(C.byref(self.desc), self.A.ctypes.data, self.noise_prec.ctypes.data,
                            self.prior_scale.ctypes.data, self.kappa2.ctypes.data,
                            self.hits.data_ptr() if self.hits is not None else None,
                            self.workspace.data_ptr(), ws, C.c_void_p(stream.cuda_stream),
                            C.byref(ctx))
        self._ctx = ctx
        if st != KCG_OK:
            msg = kcg_last_error(ctx).decode() if ctx.value else ""
            self.close()
            raise KcgError(st, msg)

    # ------------------------------------------------------------------ helpers
    def _err(self, st):
        return KcgError(st, kcg_last_error(self._ctx).decode())

    def _report(self, rep, its, hist, st) -> SolveReport:
        r = SolveReport(status=st, status_name=kcg_status_string(st).decode(),
                        converged=bool(rep.converged), iterations=rep.iterations,
                        n_systems=rep.n_systems, iterations_per=list(its[:rep.n_systems]),
                        rel_residual=rep.rel_residual, rel_residual_true=rep.rel_residual_true,
                        wall_time_s=rep.wall_time_s, loop_time_s=rep.loop_time_s,
                        system_iterations=rep.system_iterations, loop_bytes=rep.loop_bytes,
                        peak_mem_bytes=rep.peak_mem_bytes,
                        history=list(hist[:rep.history_len]) if hist is not None else [],
                        kernel_launches=rep.kernel_launches)
        return r

    def _solve(self, fn, Y, mu, tol, max_iter, n_sys, allow=(KCG_OK, KCG_NOT_CONVERGED)):
        rep = kcg_report()
        its = (C.c_int * max(n_sys, 1))()
        rep.iterations_per = C.cast(its, C.POINTER(C.c_int))
        hist = None
        if self.desc.history_cap > 0:
            hist = (C.c_double * self.desc.history_cap)()
            rep.history = C.cast(hist, C.POINTER(C.c_double))
        st = fn(self._ctx, _ptr(Y), _ptr(mu), float(tol), int(max_iter), C.byref(rep))
        if st not in allow:
            raise self._err(st)
        return self._report(rep, its, hist, st)

    def _out(self, mu, host=False):
        import torch
        if mu is not None:
            return mu
        if host:
            return torch.empty(self.shape_mu, dtype=torch.float64,
                               pin_memory=True)
        return torch.empty(self.shape_mu, dtype=torch.float64,
                           device=self.device)

    def _check_dev(self, t, shape, name):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.is_contiguous() and tuple(t.shape) == shape):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor of shape {shape}")

    def _check_host(self, a, shape, name):
        import torch
        if isinstance(a, np.ndarray):
            ok = a.dtype == np.float64 and a.flags["C_CONTIGUOUS"] and a.shape == shape
        elif isinstance(a, torch.Tensor):
            ok = (not a.is_cuda and a.dtype == torch.float64 and a.is_contiguous()
                  and tuple(a.shape) == shape)
        else:
            ok = False
        if not ok:
            raise ValueError(f"{name} must be a C-contiguous host float64 array/tensor of shape {shape}")

    # ------------------------------------------------------------------ API
    def solve(self, Y, mu=None, tol=1e-10, max_iter=100000, x0=None, **kw):
        """Kronecker route (kron_cg_solve). Y: CUDA [P][n][side][side] -> (mu, report).
        x0: optional warm start [P][k][side][side] (kron_cg_solve_x0; may be mu itself)."""
        self._check_dev(Y, self.shape_Y, "Y")
        mu = self._out(mu)
        self._check_dev(mu, self.shape_mu, "mu")
        if x0 is None:
            return mu, self._solve(kron_cg_solve, Y, mu, tol, max_iter, self.P, **kw)
        self._check_dev(x0, self.shape_mu, "x0")
        fn = lambda ctx, y, m, t, mi, rep: kron_cg_solve_x0(ctx, y, _ptr(x0), m, t, mi, rep)
        return mu, self._solve(fn, Y, mu, tol, max_iter, self.P, **kw)

    def sylvester(self, Y, mu=None, tol=1e-10, max_iter=100000, **kw):
        """Sylvester route (sylvester_solve). Y: CUDA [P][n][side][side] -> (mu, report)."""
        self._check_dev(Y, self.shape_Y, "Y")
        mu = self._out(mu)
        self._check_dev(mu, self.shape_mu, "mu")
        return mu, self._solve(sylvester_solve, Y, mu, tol, max_iter, self.P * self.k, **kw)

    def lanczos(self, Y, mu=None, tol=1e-10, max_iter=100000, **kw):
        """Block-Lanczos Sylvester solver (sylvester_lanczos_solve, Alg. SylvSolver).
        Y: CUDA [P][n][side][side] -> (mu, report); report["iterations_per"] = Lanczos steps per patch."""
        self._check_dev(Y, self.shape_Y, "Y")
        mu = self._out(mu)
        self._check_dev(mu, self.shape_mu, "mu")
        return mu, self._solve(sylvester_lanczos_solve, Y, mu, tol, max_iter, self.P, **kw)

    def kohler(self, Y, mu=None, tol=1e-10, max_iter=100000, **kw):
        """Alg. Kohler (sylvester_kohler_solve): Schur-triangular column-by-column solves."""
        self._check_dev(Y, self.shape_Y, "Y")
        mu = self._out(mu)
        self._check_dev(mu, self.shape_mu, "mu")
        return mu, self._solve(sylvester_kohler_solve, Y, mu, tol, max_iter, self.P * self.k, **kw)

    def solve_b(self, b, x=None, tol=1e-10, max_iter=100000, **kw):
        """G x = b for given right-hand sides b: CUDA [P][k][side][side] (kron_cg_solve_b)."""
        self._check_dev(b, self.shape_mu, "b")
        x = self._out(x)
        self._check_dev(x, self.shape_mu, "x")
        return x, self._solve(kron_cg_solve_b, b, x, tol, max_iter, self.P, **kw)

    def posterior_variance(self, n_probes, seed=0, var=None, tol=1e-10, max_iter=100000):
        """Hutchinson estimate of diag(G^{-1}) with n_probes Rademacher probes (posterior_variance).
        Returns (var [P][k][side][side], report)."""
        import torch
        var = self._out(var)
        self._check_dev(var, self.shape_mu, "var")
        scratch = torch.empty((2,) + self.shape_mu, dtype=torch.float64, device=self.device)
        rep = kcg_report()
        its = (C.c_int * max(self.P, 1))()
        rep.iterations_per = C.cast(its, C.POINTER(C.c_int))
        st = posterior_variance(self._ctx, int(n_probes), C.c_ulonglong(int(seed) & (2**64 - 1)), var.data_ptr(),
                                scratch.data_ptr(), float(tol), int(max_iter), C.byref(rep))
        if st not in (KCG_OK, KCG_NOT_CONVERGED):
            raise self._err(st)
        return var, self._report(rep, its, None, st)

    def solve_host(self, Y, mu=None, tol=1e-10, max_iter=100000, route="kron", **kw):
        """Host-buffer entry points (kron_cg_solve_host / sylvester_solve_host /
        sylvester_lanczos_solve_host).

        Y and mu are CPU tensors (pinned for full-speed copies) or numpy arrays: C-contiguous
        float64 of shapes shape_Y and shape_mu (checked here -- the C side copies P n N and P k N
        doubles through the raw pointers)."""
        mu = self._out(mu, host=True)
        self._check_host(Y, self.shape_Y, "Y")
        self._check_host(mu, self.shape_mu, "mu")
        fn = {"kron": kron_cg_solve_host, "sylvester": sylvester_solve_host,
              "lanczos": sylvester_lanczos_solve_host}[route]
        n_sys = self.P * self.k if route == "sylvester" else self.P
        return mu, self._solve(fn, Y, mu, tol, max_iter, n_sys, **kw)

    def solve_host_many(self, Ys, mus, tol=1e-10, max_iter=100000):
        """Pipelined host entry point (kron_cg_solve_host_many; needs host_staging=2): solve batch i
        from Ys[i] into mus[i] (pinned CPU tensors / numpy arrays) while batch i+1 is copied in and
        batch i-1 out.  Returns the list of per-batch reports."""
        nb = len(Ys)
        if nb < 1 or len(mus) != nb:
            raise ValueError("need as many outputs as inputs (>= 1)")
        for Y, mu in zip(Ys, mus):
            self._check_host(Y, self.shape_Y, "Y")
            self._check_host(mu, self.shape_mu, "mu")
        yp = (_vp * nb)(*[_ptr(Y) for Y in Ys])
        mp = (_vp * nb)(*[_ptr(mu) for mu in mus])
        reps = (kcg_report * nb)()
        its = [(C.c_int * max(self.P, 1))() for _ in range(nb)]
        for i in range(nb):
            reps[i].iterations_per = C.cast(its[i], C.POINTER(C.c_int))
        st = kron_cg_solve_host_many(self._ctx, nb, yp, mp, float(tol), int(max_iter), reps)
        if st not in (KCG_OK, KCG_NOT_CONVERGED):
            raise self._err(st)
        return [self._report(reps[i], its[i], None, reps[i].status) for i in range(nb)]

    def apply(self, x, y=None):
        """y = G x (kron_cg_apply)."""
        import torch
        shape = self.shape_mu
        self._check_dev(x, shape, "x")
        if y is None:
            y = torch.empty(shape, dtype=torch.float64, device=self.device)
        st = kron_cg_apply(self._ctx, x.data_ptr(), y.data_ptr())
        if st != KCG_OK:
            raise self._err(st)
        return y

    def rhs(self, Y, b=None):
        """b = vec(N_h Y T A) (kron_cg_rhs)."""
        import torch
        self._check_dev(Y, self.shape_Y, "Y")
        if b is None:
            b = torch.empty(self.shape_mu, dtype=torch.float64,
                            device=self.device)
        st = kron_cg_rhs(self._ctx, Y.data_ptr(), b.data_ptr())
        if st != KCG_OK:
            raise self._err(st)
        return b

    def factor(self):
        """(rho [P][k], W [P][k][k]) of Lemma 2 as computed at create (sylvester_factor)."""
        rho = np.empty((self.P, self.k))
        W = np.empty((self.P, self.k, self.k))
        st = sylvester_factor(self._ctx, rho.ctypes.data, W.ctypes.data)
        if st != KCG_OK:
            raise self._err(st)
        return rho, W

    def launch_config(self) -> dict:
        """Diagnostic: CG-kernel grid / dynamic smem per route and the device SM count
        (kcg_debug_config, not part of the ABI header)."""
        f = _lib.kcg_debug_config
        f.restype, f.argtypes = C.c_int, [_ctxp, C.c_void_p]
        out = (C.c_longlong * 8)()
        f(self._ctx, out)
        return dict(grid_kron=out[0], grid_syl=out[1], smem_kron=out[2], smem_syl=out[3], sm_count=out[4],
                    resident_kron=out[5], resident_syl=out[6], resident_kohler=out[7])

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            kron_cg_destroy(self._ctx)
        self._ctx = _ctxp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass



# ------------------------------------------------------------------------------ row slabs
def slab_rows(level: int, nranks: int) -> int:
    """Rows of each rank's slab when a 2^level face is split over nranks ranks."""
    side = 1 << level
    if nranks < 1 or nranks > 8 or side % nranks or side // nranks < 4:
        raise ValueError(f"cannot split a {side}-row face into {nranks} slabs of >= 4 rows")
    return side // nranks


def split_rows(a, nranks: int):
    """[..., side, side] -> [nranks, ..., rows, side] (contiguous): rank r gets rows [r rows, (r+1) rows)."""
    side = a.shape[-2]
    rows = side // nranks
    parts = [a[..., r * rows:(r + 1) * rows, :] for r in range(nranks)]
    import torch
    if isinstance(a, torch.Tensor):
        return torch.stack(parts).contiguous()
    return np.ascontiguousarray(np.stack(parts))


def join_rows(parts):
    """Inverse of split_rows: [nranks, ..., rows, side] -> [..., nranks rows, side]."""
    import torch
    if isinstance(parts, torch.Tensor):
        return torch.cat(list(parts), dim=-2)
    return np.concatenate(list(parts), axis=-2)


def ghost_rows(a, nranks: int, ghost: int):
    """[..., side, side] -> [nranks, ..., rows + 2 ghost, side]: each rank's slab with `ghost` rows of
    the face above and below (zeros beyond the face) -- the layout of slab hits maps."""
    import torch
    side = a.shape[-2]
    rows = side // nranks
    pad = torch.zeros(a.shape[:-2] + (ghost, a.shape[-1]), dtype=a.dtype, device=a.device)
    full = torch.cat([pad, a, pad], dim=-2)
    return torch.stack([full[..., r * rows:r * rows + rows + 2 * ghost, :] for r in range(nranks)]).contiguous()


def ipc_export(t) -> bytes:
    """72-byte record (CUDA IPC handle of the allocation + offset) naming device tensor t for peers."""
    h = C.create_string_buffer(64)
    off = C.c_size_t()
    st = kcg_ipc_export(t.data_ptr(), h, C.byref(off))
    if st != KCG_OK:
        raise KcgError(st, "kcg_ipc_export")
    return h.raw + int(off.value).to_bytes(8, "little")


def ipc_import(rec: bytes):
    """(device pointer, mapping base) of a peer's ipc_export record."""
    ptr, base = _vp(), _vp()
    st = kcg_ipc_import(rec[:64], int.from_bytes(rec[64:72], "little"), C.byref(ptr), C.byref(base))
    if st != KCG_OK:
        raise KcgError(st, "kcg_ipc_import")
    return ptr.value, base.value


def exchange_records(rec: bytes, group=None) -> list:
    """All-gather one fixed-size byte record per rank over a torch.distributed group (host logic
    of the slab set-up; works on gloo and nccl)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.frombuffer(bytearray(rec), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [bytes(o.cpu().numpy().tobytes()) for o in out]


class KronCGSlab(KronCG):
    """Row-slab context: every face split over `nranks` ranks (kron_cg_create_slab).

    emulate=True: this process drives all ranks on one GPU (one cooperative launch; the layout of
    Y / mu is [nranks][P][..][rows][side]; hits is given for the whole face [P][side][side]).  emulate=False: this process is rank
    `dist.get_rank(group)` of `group`; workspaces are exchanged through CUDA IPC and Y / mu are
    [1][P][..][rows][side] (its own slab).
    """

    def __init__(self, level, A, noise_prec, prior_scale, kappa2, nranks, emulate=True, group=None,
                 hits=None, device=None, host_staging=False, history_cap=0, stream=None,
                 precond="none"):
        import torch
        A = np.ascontiguousarray(np.asarray(A, dtype=np.float64))
        if A.ndim == 2:
            A = A[None]
        P, n, k = A.shape
        self.noise_prec = np.ascontiguousarray(np.asarray(noise_prec, dtype=np.float64).reshape(P, n))
        self.prior_scale = np.ascontiguousarray(np.asarray(prior_scale, dtype=np.float64).reshape(P, k))
        self.kappa2 = np.ascontiguousarray(np.asarray(kappa2, dtype=np.float64).reshape(P))
        self.A = A
        self.level, self.P, self.n, self.k = level, P, n, k
        self.side = 1 << level
        self.nranks = nranks
        self.rows = slab_rows(level, nranks)
        self.N = self.rows * self.side
        self.device = torch.device(device if device is not None else "cuda")
        self._ipc_bases = []
        if emulate:
            self.rank0, self.nlocal = 0, nranks
        else:
            import torch.distributed as dist
            if dist.get_world_size(group) != nranks:
                raise ValueError("group size must equal nranks")
            self.rank0, self.nlocal = dist.get_rank(group), 1
        self.shape_Y = (self.nlocal, P, n, self.rows, self.side)
        self.shape_mu = (self.nlocal, P, k, self.rows, self.side)
        pc = {"none": KCG_PRECOND_NONE, "block_jacobi": KCG_PRECOND_BLOCK_JACOBI}[precond]
        self.desc = kcg_desc(level, n, k, P, KCG_PRIOR_LAPLACIAN, KCG_LAYOUT_ROW_MAJOR,
                             pc, int(bool(host_staging)), int(history_cap))
        ws = kron_cg_workspace_size_slab(C.byref(self.desc), nranks)
        if ws == 0:
            raise KcgError(KCG_E_SHAPE, "invalid descriptor or slab split")
        self.ws_bytes = ws
        sl = kcg_slab()
        sl.nranks, sl.rank0, sl.nlocal = nranks, self.rank0, self.nlocal
        self.workspaces = [torch.empty(ws + 256, dtype=torch.uint8, device=self.device)
                           for _ in range(self.nlocal)]
        own = [w.data_ptr() + (-w.data_ptr()) % 256 for w in self.workspaces]
        if emulate:
            for r in range(nranks):
                sl.peer_ws[r] = own[r]
        else:
            # the workspace allocation is exported whole; the record carries the aligned offset
            rec = ipc_export(self.workspaces[0])
            rec = rec[:64] + (int.from_bytes(rec[64:72], "little") + own[0] - self.workspaces[0].data_ptr()).to_bytes(8, "little")
            recs = exchange_records(rec, group)
            for r in range(nranks):
                if r == self.rank0:
                    sl.peer_ws[r] = own[0]
                else:
                    ptr, base = ipc_import(recs[r])
                    self._ipc_bases.append(base)
                    sl.peer_ws[r] = ptr
        self.hits = None
        if hits is not None:  # full-face hits [P][side][side] -> ghosted slabs of the local ranks
            self.hits = ghost_rows(hits.to(dtype=torch.float64), nranks, 2)[self.rank0:self.rank0 + self.nlocal]
            self.hits = self.hits.to(device=self.device).contiguous()
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        ctx = _ctxp()
        st = kron_cg_create_slab(C.byref(self.desc), C.byref(sl), self.A.ctypes.data,
                                 self.noise_prec.ctypes.data, self.prior_scale.ctypes.data,
                                 self.kappa2.ctypes.data,
                                 self.hits.data_ptr() if self.hits is not None else None,
                                 ws, C.c_void_p(stream.cuda_stream), C.byref(ctx))
        self._ctx = ctx
        if st != KCG_OK:
            msg = kcg_last_error(ctx).decode() if ctx.value else ""
            self.close()
            raise KcgError(st, msg)
        if not emulate:
            import torch.distributed as dist
            dist.barrier(group)  # every rank's context (zeroed flags, ghost rows) exists before solves

    def probe_put(self, value: float):
        """Diagnostic: peer-store value + rank into every rank's probe slot (kcg_slab_probe_put)."""
        st = kcg_slab_probe_put(self._ctx, float(value))
        if st != KCG_OK:
            raise self._err(st)

    def probe_get(self) -> list:
        """Diagnostic: this process's probe slots of all ranks (kcg_slab_probe_get)."""
        out = (C.c_double * self.nranks)()
        st = kcg_slab_probe_get(self._ctx, out)
        if st != KCG_OK:
            raise self._err(st)
        return list(out)

    def close(self):
        super().close()
        for b in getattr(self, "_ipc_bases", []):
            kcg_ipc_close(b)
        self._ipc_bases = []
