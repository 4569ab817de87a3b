"""Oracle: the paper's Alg. Kohler (sparse-dense Sylvester solver) step by step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  For Eq.(Axb-Sylv) P:L263-265 with the general
prior block Q0 (reading R3): H = N_h^{-1} Q0, S = S^ = A^T T A P^{-1}, F = Y^ = Y T A P^{-1}.
  1. Schur decomposition S = W R W^T, W^T W = I, R upper triangular.
  2. F^ := F W.
  3. for i = 1..m:  F^_i := F^_i - sum_{k<i} X^_k R_ki;  solve (H + R_ii I) X^_i = F^_i.
  4. X := X^ W^T.
Readings (R33): the algorithm box prints "F^ := F_i - ..." and "X := X^ W"; with
S = W R W^T the algebra (H X + X S = F  <=>  H (X W) + (X W) R = F W) gives the i-th column of F^ and
X = X^ W^T.  Which Schur form: S^ has real eigenvalues (Lemma 2), so its real Schur form is
triangular; the canonical one used here (and by the GPU) orders the eigenvalues ascending on R's
diagonal and takes W = the Q factor (positive diagonal of the triangular factor) of the Lemma-2
eigenvectors U = P W_eig in that order, so W^T S W = T diag(rho) T^{-1} is upper triangular.
Each column solve uses the symmetric form (Q0 + R_ii N_h) X^_i = N_h F^_i (reading R14) with the
oracle CG, stop on ||r_i|| <= tol ||N_h F^_i|| (reading R15).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import cg as cg_mod
from . import grid, model
from .sylvester import small_factor


@dataclass
class KohlerResult:
    x: np.ndarray          # vec(X), component-major (m N,)
    iterations: list       # per column
    converged: bool
    W: np.ndarray          # orthogonal Schur vectors
    R: np.ndarray          # upper triangular Schur factor


def schur_factor(A, noise_prec, tau):
    """(S^, W, R): the canonical real Schur decomposition S^ = W R W^T described above."""
    M, P, rho, We = small_factor(A, noise_prec, tau)
    S = M @ np.linalg.inv(P)
    U = P @ We                                  # S^ U = U diag(rho), ascending
    Q, T = np.linalg.qr(U)
    d = np.sign(np.diag(T))
    d[d == 0] = 1.0
    W = Q * d[None, :]                          # positive diagonal of the triangular factor
    R = W.T @ S @ W
    return S, W, R


def solve(level, A, noise_prec, tau, kappa2, Y, hits=None, prior="laplacian", tol=1e-10,
          max_iter=100000) -> KohlerResult:
    A = np.asarray(A, dtype=np.float64)
    n, m = A.shape
    N = grid.side_of(level) ** 2
    h = model._hits_vec(level, hits)
    Q0 = model.prior_Q0(level, kappa2, prior)
    S, W, R = schur_factor(A, noise_prec, tau)
    P = np.diag(np.asarray(tau, dtype=np.float64))
    Ymaps = np.asarray(Y, dtype=np.float64).reshape(n, N).T
    F = Ymaps @ np.diag(np.asarray(noise_prec, dtype=np.float64)) @ A @ np.linalg.inv(P)   # Y^
    Fh = F @ W                                   # F^ := F W
    Xh = np.zeros((N, m))
    its, ok = [], True
    for i in range(m):
        f = Fh[:, i] - sum(Xh[:, k] * R[k, i] for k in range(i)) if i > 0 else Fh[:, i]
        H = (Q0 + R[i, i] * sp.diags(h)).tocsr()   # symmetric form of (H + R_ii I)
        res = cg_mod.cg_hs(H, h * f, tol=tol, max_iter=max_iter)
        Xh[:, i] = res.x
        its.append(res.iterations)
        ok = ok and res.converged
    X = Xh @ W.T                                 # X := X^ W^T
    return KohlerResult(X.T.reshape(-1).copy(), its, ok, W, R)


def problem_solve(p, tol=1e-10, max_iter=100000) -> KohlerResult:
    return solve(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.Y, p.hits, p.prior, tol=tol, max_iter=max_iter)
