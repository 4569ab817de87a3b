"""Oracle: the Sylvester route, diagonalised into k decoupled shifted systems.

PAPER.md:
  * Sec. 3.3 P:L252-265 -- reshaping Eq.(Axb) gives the generalised Sylvester equation
    D^2 M P + N M A^T T A = N Y T A  (here with the general prior block Q0 in place of
    D^2, reading R3), i.e. Q0 X P + N_h X M = F with M = A^T T A, F = reshape(b, N, k).
  * Alg.Kohler P:L279-291 -- transform the small factor, solve shifted systems
    (H + R_ii I) X_i = F_i column by column, transform back.
  * Lemma 2 P:L436-453 -- S^ = A^T T A P^{-1} is self-adjoint in <.,.>_{P^{-1}}, hence
    diagonalisable: S^ = U R U^{-1}, U^T P^{-1} U = I, computed once.
Reading R13/R14: with (rho, W) = eigh(M, P) (ascending rho, W^T P W = I, U = P W) the
Schur factor R is diagonal, so the Kohler back-substitution sum vanishes and the
column systems decouple:  (Q0 + rho_i N_h) xt_i = ft_i  with  Ft = F W,  X = Xt W^T.
The symmetric form (Q0 + rho_i N_h) is used instead of N^{-1} Q0 + rho_i I (same
solution, SPD in the Euclidean inner product).  Reading R15: each column stops on
||rt_i|| <= tol ||ft_i||.  Sign convention of W: the largest-magnitude entry of every
column is positive.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import cg as cg_mod
from . import grid, model


@dataclass
class SylvesterResult:
    x: np.ndarray            # vec(X), component-major (k*N,)
    iterations: list         # per column
    converged: bool
    rho: np.ndarray
    W: np.ndarray
    col_rel_residual: list


def small_factor(A, noise_prec, tau):
    """M = A^T T A, P = diag(phi), and the generalised eigenpairs of (M, P) (Lemma 2)."""
    A = np.asarray(A, dtype=np.float64)
    M = A.T @ np.diag(np.asarray(noise_prec, dtype=np.float64)) @ A
    P = np.diag(np.asarray(tau, dtype=np.float64))
    rho, W = sla.eigh(M, P)               # ascending; W^T P W = I
    for i in range(W.shape[1]):
        c = W[:, i]
        if c[np.argmax(np.abs(c))] < 0:
            W[:, i] = -c
    return M, P, rho, W


def solve(level, A, noise_prec, tau, kappa2, Y, hits=None, prior="laplacian",
          tol=1e-10, max_iter=100000, precond=None) -> SylvesterResult:
    """precond=None (the paper's CG) or "jacobi": z = r / diag(Q0 + rho_i N_h) -- the k = 1 case of
    the pixel-block Jacobi option (reading R10)."""
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    N = grid.side_of(level) ** 2
    M, P, rho, W = small_factor(A, noise_prec, tau)
    b = model.assemble_rhs(level, A, noise_prec, Y, hits)
    F = b.reshape(k, N).T                 # reshape(b, N, k): column l = component l
    Ft = F @ W                            # F^ := F W
    Q0 = model.prior_Q0(level, kappa2, prior)
    h = np.ones(N) if hits is None else np.asarray(hits, dtype=np.float64).reshape(N)
    Xt = np.zeros((N, k))
    its, rels, ok = [], [], True
    for i in range(k):
        H = (Q0 + rho[i] * sp.diags(h)).tocsr()      # (Q0 + rho_i N_h)
        pc = None
        if precond == "jacobi":
            dH = H.diagonal().copy()
            pc = lambda r, dH=dH: r / dH
        res = cg_mod.cg_hs(H, Ft[:, i], tol=tol, max_iter=max_iter, precond=pc)
        Xt[:, i] = res.x
        its.append(res.iterations)
        rels.append(res.rel_residual)
        ok = ok and res.converged
    X = Xt @ W.T                          # X := X^ W^T
    return SylvesterResult(X.T.reshape(-1).copy(), its, ok, rho, W, rels)


def problem_solve(p, tol=1e-10, max_iter=100000, precond=None) -> SylvesterResult:
    return solve(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.Y, p.hits, p.prior,
                 tol=tol, max_iter=max_iter, precond=precond)
