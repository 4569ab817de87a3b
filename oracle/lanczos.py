"""Oracle: the paper's block-Lanczos Sylvester solver (Alg. SylvSolver).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): plain numpy, fp64, step by step in the
paper's order and notation; no blocking or fusion.

PAPER.md:
  * Eq.(Axb-Sylv) P:L263-265 -- N^{-1} D^2 M + M A^T T A P^{-1} = Y T A P^{-1}; here with the
    general prior block Q0 (reading R3) and the hit counts N_h: the large coefficient
    AA := N_h^{-1} Q0, the small one S^ := A^T T A P^{-1}, the right-hand side Y^ := Y T A P^{-1}
    (N x m, columns = components; Y is N x n, pixels by maps).
  * Lemma 1 P:L317-327 -- AA is symmetric in (x, y)_N = y^T N_h x, so block Lanczos in that inner
    product has a three-term recurrence (Alg. Lanczos).
  * Eq.(Sylv-small) P:L430 -- Galerkin projection T_j Z_j + Z_j S^ = E_1 B_0.
  * Lemma 2 P:L436-453 -- S^ = U R U^{-1}, U^T P^{-1} U = I.
  * Eq.(soln-constr) P:L484-486 -- Z_j = Q_j F_j U^T P^{-1}, F_kl = (Q_j^T E_1 B_0 U)_kl / (phi_k + rho_l).
  * Alg. SylvSolver P:L500-570 -- residual estimate gamma, stop when sqrt(gamma) <= eps ||B_0||_F,
    then rerun Lanczos with the stored coefficients to assemble M = sum_j V_j G_j.
Readings (R25-R28):
  R25 the recurrence is W = AA V_i - V_{i-1} B_i^T (T_j symmetric: sub-diagonal B, super-diagonal
      B^T; the paper prints B in both places);
  R26 "Q_i E_m" in gamma is the last block ROW of Q_i (E_m^T Q_i), i.e. gamma = ||B_{i+1} E_m^T Q_i F||_F^2;
  R27 Z = Q F U^{-1} = Q F U^T P^{-1} (Eq.(soln-constr); the algorithm box drops P^{-1});
  R28 QR in (.,.)_N by Cholesky: C = W^T N_h W = R^T R, B = R (upper), V = W B^{-1}.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import grid, model
from .sylvester import small_factor


@dataclass
class LanczosResult:
    x: np.ndarray                 # vec(M): component-major (k*N,)
    iterations: int
    converged: bool
    gamma_history: list = field(default_factory=list)   # sqrt(gamma) / ||B_0||_F per iteration
    H: list = field(default_factory=list)               # H_i (m x m)
    B: list = field(default_factory=list)               # B_0, B_2, ..., B_{i+1} (m x m, upper)
    V: list = field(default_factory=list)               # V_1, V_2, ... (kept only if keep_basis)


def n_qr(W: np.ndarray, h: np.ndarray):
    """QR factorization in (.,.)_N (reading R28): W = V B, V^T N V = I, B upper triangular."""
    C = W.T @ (h[:, None] * W)
    R = np.linalg.cholesky(C).T            # C = R^T R
    return np.linalg.solve(R.T, W.T).T, R  # V = W R^{-1}


def solve(level, A, noise_prec, tau, kappa2, Y, hits=None, prior="laplacian", tol=1e-10, max_iter=1000,
          keep_basis=False) -> LanczosResult:
    A = np.asarray(A, dtype=np.float64)
    n, m = A.shape
    N = grid.side_of(level) ** 2
    h = model._hits_vec(level, hits)
    Q0 = model.prior_Q0(level, kappa2, prior)
    AA = lambda V: (Q0 @ V) / h[:, None]                        # N_h^{-1} Q0 V
    Mk, P, rho, W_eig = small_factor(A, noise_prec, tau)        # M = A^T T A, P = diag(phi)
    U = P @ W_eig                                               # S^ = U R U^{-1}, U^T P^{-1} U = I
    Uinv = U.T @ np.linalg.inv(P)
    Ymaps = np.asarray(Y, dtype=np.float64).reshape(n, N).T     # N x n
    Yhat = Ymaps @ np.diag(np.asarray(noise_prec, dtype=np.float64)) @ A @ np.linalg.inv(P)   # Y T A P^{-1}
    V, B0 = n_qr(Yhat, h)                                       # Y^ = V_1 B_0
    nB0 = np.linalg.norm(B0)
    res = LanczosResult(np.zeros(m * N), 0, False, [], [], [B0], [])
    if nB0 == 0.0:
        res.converged = True
        return res
    V_old = np.zeros_like(V)
    Hs, Bs = [], [B0]
    i = 0
    while i < max_iter:
        i += 1
        if keep_basis:
            res.V.append(V.copy())
        # Lanczos step (Alg. Lanczos / SylvSolver)
        W = AA(V)
        if i > 1:
            W = W - V_old @ Bs[-1].T
        H = V.T @ (h[:, None] * W)
        W = W - V @ H
        V_old = V
        V, Bn = n_qr(W, h)
        Hs.append(H)
        Bs.append(Bn)
        # residual norm estimate: eigendecomposition of T_i
        T = np.zeros((i * m, i * m))
        for a in range(i):
            T[a * m:(a + 1) * m, a * m:(a + 1) * m] = Hs[a]
            if a + 1 < i:
                T[(a + 1) * m:(a + 2) * m, a * m:(a + 1) * m] = Bs[a + 1]
                T[a * m:(a + 1) * m, (a + 1) * m:(a + 2) * m] = Bs[a + 1].T
        phi, Qm = np.linalg.eigh(T)
        S = (U.T @ B0.T) @ Qm[:m, :]                           # (U^T B_0^T)(E_1^T Q_i)
        J = Qm[-m:, :].T @ Bn.T                                 # (E_m^T Q_i)^T B_{i+1}^T   (R26)
        gamma = 0.0
        for j in range(m):
            Kd = rho[j] + phi                                   # K = rho_j I + Phi_i
            gamma += float(np.sum(((S[j, :] / Kd) @ J) ** 2))
        res.gamma_history.append(np.sqrt(gamma) / nB0)
        if np.sqrt(gamma) <= tol * nB0:
            res.converged = True
            break
    # construct the coefficients (Eq.(soln-constr), R27)
    E1B0U = np.zeros((i * m, m))
    E1B0U[:m, :] = B0 @ U
    F = (Qm.T @ E1B0U) / (phi[:, None] + rho[None, :])
    Z = Qm @ F @ Uinv
    # rerun Lanczos with the stored coefficients to assemble M = sum_j V_j G_j
    Mx = np.zeros((N, m))
    V = np.linalg.solve(B0.T, Yhat.T).T                         # Y^ B_0^{-1}, as n_qr formed V_1 (R30)
    V_old = np.zeros_like(V)
    for j in range(1, i + 1):
        Mx += V @ Z[(j - 1) * m:j * m, :]
        W = AA(V)
        if j > 1:
            W = W - V_old @ Bs[j - 1].T
        W = W - V @ Hs[j - 1]
        V_old = V
        V = np.linalg.solve(Bs[j].T, W.T).T                    # W B_{j+1}^{-1}
    res.x = Mx.T.reshape(-1).copy()
    res.iterations = i
    res.H, res.B = Hs, Bs
    return res


def problem_solve(p, tol=1e-10, max_iter=1000, keep_basis=False) -> LanczosResult:
    return solve(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.Y, p.hits, p.prior, tol=tol, max_iter=max_iter,
                 keep_basis=keep_basis)
