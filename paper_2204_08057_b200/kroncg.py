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
KCG_E_NONFINITE, KCG_E_BREAKDOWN, KCG_E_CUDA, KCG_E_NCCL, KCG_E_STATE = 5, 6, 7, 8, 9
KCG_PRIOR_LAPLACIAN, KCG_PRIOR_D2 = 0, 1
KCG_LAYOUT_ROW_MAJOR, KCG_LAYOUT_NESTED = 0, 1
KCG_PRECOND_NONE, KCG_PRECOND_BLOCK_JACOBI = 0, 1


class kcg_desc(C.Structure):
    _fields_ = [("level", C.c_int), ("n_freq", C.c_int), ("n_comp", C.c_int),
                ("n_patches", C.c_int), ("prior", C.c_int), ("layout", C.c_int),
                ("precond", C.c_int), ("host_staging", C.c_int), ("history_cap", C.c_int)]


class kcg_report(C.Structure):
    _fields_ = [("status", C.c_int), ("converged", C.c_int), ("iterations", C.c_int),
                ("n_systems", C.c_int), ("iterations_per", C.POINTER(C.c_int)),
                ("rel_residual", C.c_double), ("rel_residual_true", C.c_double),
                ("wall_time_s", C.c_double), ("loop_time_s", C.c_double),
                ("system_iterations", C.c_longlong), ("loop_bytes", C.c_double),
                ("peak_mem_bytes", C.c_size_t), ("history", C.POINTER(C.c_double)),
                ("history_len", C.c_int)]


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
kron_cg_apply = _sig("kron_cg_apply", C.c_int, [_ctxp, _vp, _vp])
kron_cg_rhs = _sig("kron_cg_rhs", C.c_int, [_ctxp, _vp, _vp])
sylvester_factor = _sig("sylvester_factor", C.c_int, [_ctxp, _vp, _vp])
kcg_last_error = _sig("kcg_last_error", C.c_char_p, [_ctxp])
kcg_status_string = _sig("kcg_status_string", C.c_char_p, [C.c_int])
kron_cg_destroy = _sig("kron_cg_destroy", None, [_ctxp])

EXPORTS = ["kron_cg_workspace_size", "kron_cg_create", "kron_cg_solve", "sylvester_solve",
           "kron_cg_solve_host", "sylvester_solve_host", "kron_cg_apply", "kron_cg_rhs",
           "sylvester_factor", "kcg_last_error", "kcg_status_string", "kron_cg_destroy"]


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
    """

    def __init__(self, level, A, noise_prec, prior_scale, kappa2, hits=None, device=None,
                 host_staging=False, history_cap=0, stream=None, precond="none"):
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
        pc = {"none": KCG_PRECOND_NONE, "block_jacobi": KCG_PRECOND_BLOCK_JACOBI}[precond]
        self.desc = kcg_desc(level, n, k, P, KCG_PRIOR_LAPLACIAN, KCG_LAYOUT_ROW_MAJOR,
                             pc, int(bool(host_staging)), int(history_cap))
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
                        history=list(hist[:rep.history_len]) if hist is not None else [])
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
            return torch.empty((self.P, self.k, self.side, self.side), dtype=torch.float64,
                               pin_memory=True)
        return torch.empty((self.P, self.k, self.side, self.side), dtype=torch.float64,
                           device=self.device)

    def _check_dev(self, t, shape, name):
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.is_contiguous() and tuple(t.shape) == shape):
            raise ValueError(f"{name} must be a contiguous CUDA float64 tensor of shape {shape}")

    # ------------------------------------------------------------------ API
    def solve(self, Y, mu=None, tol=1e-10, max_iter=100000, **kw):
        """Kronecker route (kron_cg_solve). Y: CUDA [P][n][side][side] -> (mu, report)."""
        self._check_dev(Y, (self.P, self.n, self.side, self.side), "Y")
        mu = self._out(mu)
        self._check_dev(mu, (self.P, self.k, self.side, self.side), "mu")
        return mu, self._solve(kron_cg_solve, Y, mu, tol, max_iter, self.P, **kw)

    def sylvester(self, Y, mu=None, tol=1e-10, max_iter=100000, **kw):
        """Sylvester route (sylvester_solve). Y: CUDA [P][n][side][side] -> (mu, report)."""
        self._check_dev(Y, (self.P, self.n, self.side, self.side), "Y")
        mu = self._out(mu)
        self._check_dev(mu, (self.P, self.k, self.side, self.side), "mu")
        return mu, self._solve(sylvester_solve, Y, mu, tol, max_iter, self.P * self.k, **kw)

    def solve_host(self, Y, mu=None, tol=1e-10, max_iter=100000, route="kron", **kw):
        """Host-buffer entry points (kron_cg_solve_host / sylvester_solve_host).

        Y and mu are CPU tensors (pinned for full-speed copies) or numpy arrays."""
        mu = self._out(mu, host=True)
        fn = kron_cg_solve_host if route == "kron" else sylvester_solve_host
        n_sys = self.P if route == "kron" else self.P * self.k
        return mu, self._solve(fn, Y, mu, tol, max_iter, n_sys, **kw)

    def apply(self, x, y=None):
        """y = G x (kron_cg_apply)."""
        import torch
        shape = (self.P, self.k, self.side, self.side)
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
        self._check_dev(Y, (self.P, self.n, self.side, self.side), "Y")
        if b is None:
            b = torch.empty((self.P, self.k, self.side, self.side), dtype=torch.float64,
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
        out = (C.c_longlong * 5)()
        f(self._ctx, out)
        return dict(grid_kron=out[0], grid_syl=out[1], smem_kron=out[2], smem_syl=out[3], sm_count=out[4])

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            kron_cg_destroy(self._ctx)
        self._ctx = _ctxp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
