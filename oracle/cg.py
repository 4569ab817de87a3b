"""Oracle: conjugate gradients on the assembled Kronecker system.

PAPER.md Sec. 3.2 P:L225-241 presents CG for G = Q + B^T C B and b = B^T C Y as
Algorithm \\CGnoprecond, whose body is an unexpanded macro -- reading R7:
the textbook Hestenes-Stiefel CG of the paper's cited reference (Saad, Iterative
Methods for Sparse Linear Systems, Alg. 6.18), with x0 = 0 and the stopping rule of
reading R8: stop after the first iteration j with ||r_j||_2 <= tol * ||b||_2;
"iterations" = number of x-updates.  ||b|| = 0 returns x = 0 after 0 iterations.

Also here: the single-pass (Chronopoulos-Gear) CG variant that the GPU kernel runs
(reading R9: the paper's "two variants of the CG approach"), written
step by step in the same notation so GPU and oracle can be compared like-for-like.
Both accept an optional preconditioner solve z = K^{-1} r ("preconditioning
techniques can be used"; default none, as in the paper).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class CGResult:
    x: np.ndarray
    iterations: int
    converged: bool
    rel_residual: float          # recursive ||r_j|| / ||b||
    history: list = field(default_factory=list)
    status: str = "ok"           # ok | not_converged | breakdown | nonfinite


def cg_hs(G, b, tol=1e-10, max_iter=10000, precond=None, callback=None, x0=None) -> CGResult:
    """Textbook (preconditioned) Hestenes-Stiefel CG (Saad Alg. 6.18 / 9.1), x0 = 0 by default.

    x0 given (warm start, reading R37): Saad's r_0 = b - A x_0; the stopping rule stays
    ||r_j|| <= tol ||b|| (||r_0|| when b = 0), tested before the first step too (x_0 may already
    satisfy it: 0 iterations)."""
    b = np.asarray(b, dtype=np.float64)
    bnorm = float(np.sqrt(b @ b))
    if x0 is None:
        x = np.zeros_like(b)
        if bnorm == 0.0:
            return CGResult(x, 0, True, 0.0, [])
        r = b.copy()
    else:
        x = np.array(x0, dtype=np.float64).reshape(b.shape)
        r = b - G @ x
        r0 = float(np.sqrt(r @ r))
        if bnorm == 0.0:
            bnorm = r0
        if r0 <= tol * bnorm:
            return CGResult(x, 0, True, r0 / bnorm if bnorm > 0 else 0.0, [])
    z = r if precond is None else precond(r)
    p = z.copy()
    rz = float(r @ z)
    hist = []
    for j in range(1, max_iter + 1):
        q = G @ p                      # q = G p
        pq = float(p @ q)
        if not np.isfinite(pq):
            return CGResult(x, j - 1, False, hist[-1] if hist else 1.0, hist, "nonfinite")
        if pq <= 0.0:
            return CGResult(x, j - 1, False, hist[-1] if hist else 1.0, hist, "breakdown")
        alpha = rz / pq                # alpha_j = (r, z) / (p, G p)
        x = x + alpha * p              # x_{j+1} = x_j + alpha p_j
        r = r - alpha * q              # r_{j+1} = r_j - alpha G p_j
        rnorm = float(np.sqrt(r @ r))
        hist.append(rnorm / bnorm)
        if callback is not None:
            callback(j, x, r)
        if rnorm <= tol * bnorm:
            return CGResult(x, j, True, rnorm / bnorm, hist)
        z = r if precond is None else precond(r)
        rz_new = float(r @ z)
        beta = rz_new / rz             # beta_j = (r_{j+1}, z_{j+1}) / (r_j, z_j)
        p = z + beta * p               # p_{j+1} = z_{j+1} + beta p_j
        rz = rz_new
    return CGResult(x, max_iter, False, hist[-1], hist, "not_converged")


def cg_single_pass(G, b, tol=1e-10, max_iter=10000, precond=None) -> CGResult:
    """Single-reduction CG (Chronopoulos & Gear 1989), x0 = 0.

    Per iteration i, with scalars alpha_i, beta_i known:
        p_i = u_i + beta_i p_{i-1}
        s_i = G p_i                   (recomputed, not recurred)
        x_{i+1} = x_i + alpha_i p_i
        r_{i+1} = r_i - alpha_i s_i
        u_{i+1} = K^{-1} r_{i+1};  w_{i+1} = G u_{i+1}
        gamma_{i+1} = (r_{i+1}, u_{i+1});  delta_{i+1} = (w_{i+1}, u_{i+1})
        beta_{i+1} = gamma_{i+1} / gamma_i
        alpha_{i+1} = gamma_{i+1} / (delta_{i+1} - beta_{i+1} gamma_{i+1} / alpha_i)
    Start: r_0 = b, u_0 = K^{-1} b, w_0 = G u_0, alpha_0 = gamma_0 / delta_0, beta_0 = 0.
    Convergence is tested on ||r_{i+1}||_2 (reading R8), so the iteration count has the
    same meaning as cg_hs.
    """
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    bnorm = float(np.sqrt(b @ b))
    if bnorm == 0.0:
        return CGResult(x, 0, True, 0.0, [])
    M = (lambda v: v) if precond is None else precond
    r = b.copy()
    u = M(r)
    w = G @ u
    gamma = float(r @ u)
    delta = float(w @ u)
    if delta <= 0.0:
        return CGResult(x, 0, False, 1.0, [], "breakdown")
    alpha = gamma / delta
    beta = 0.0
    p = np.zeros_like(b)
    hist = []
    for i in range(max_iter):
        p = u + beta * p
        s = G @ p
        x = x + alpha * p
        r = r - alpha * s
        u = M(r)
        w = G @ u
        gamma_new = float(r @ u)
        delta = float(w @ u)
        rnorm = float(np.sqrt(r @ r))
        hist.append(rnorm / bnorm)
        if not (np.isfinite(gamma_new) and np.isfinite(delta)):
            return CGResult(x, i + 1, False, hist[-1], hist, "nonfinite")
        if rnorm <= tol * bnorm:
            return CGResult(x, i + 1, True, rnorm / bnorm, hist)
        beta = gamma_new / gamma
        den = delta - beta * gamma_new / alpha
        if den <= 0.0:
            return CGResult(x, i + 1, False, hist[-1], hist, "breakdown")
        alpha = gamma_new / den
        gamma = gamma_new
    return CGResult(x, max_iter, False, hist[-1], hist, "not_converged")


def block_jacobi_precond(level, A, noise_prec, tau, kappa2, hits=None, prior="laplacian"):
    """Pixel-block Jacobi K_j = h_j M + diag(Q0)_jj P  (reading R10; an option, not the paper's).

    Returns z = K^{-1} r acting on component-major vectors (k*N,).  K_j is the k x k
    diagonal block of G at pixel j, taken from the assembled matrix.
    """
    from . import model
    G = model.assemble_G(level, A, noise_prec, tau, kappa2, hits, prior)
    k = np.asarray(A).shape[1]
    N = G.shape[0] // k
    blocks = np.empty((N, k, k))
    Gc = G.tocsc()
    for a in range(k):
        for c in range(k):
            sub = Gc[a * N:(a + 1) * N, c * N:(c + 1) * N]
            blocks[:, a, c] = sub.diagonal()
    inv = np.linalg.inv(blocks)

    def apply(r):
        R = r.reshape(k, N).T           # (N, k)
        Z = np.einsum("jab,jb->ja", inv, R)
        return Z.T.reshape(-1).copy()

    return apply
