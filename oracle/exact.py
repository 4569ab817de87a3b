"""Oracle: exact references for mu* = G^{-1} b (Eq.(mu*) P:L78-82; G SPD).

dense_solve  -- explicit dense G and a Cholesky solve (SPEC dense_oracle S:L419-453),
                guarded to m*N <= 8192.
dct_exact    -- mode-wise exact solve when all hit counts are 1: the free-boundary face
                Laplacian L is diagonalised by the orthonormal 2-D DCT-II with eigenvalues
                lam_ab = (2 - 2cos(pi a/s)) + (2 - 2cos(pi b/s)) (textbook Neumann-grid
                spectrum), and D^2 = L^2 by lam_ab^2.  Since G = M (x) I + P (x) Q0
                (P:L147), each DCT mode (a, b) decouples into the k x k system
                (M + lam^{Q0}_ab P) xhat_ab = fhat_ab.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
from scipy.fft import dctn, idctn

from . import grid, model

DENSE_GUARD = 8192


def dense_solve(G, b) -> np.ndarray:
    """Direct Cholesky solve of the assembled system (test oracle only)."""
    if G.shape[0] > DENSE_GUARD:
        raise MemoryError(f"dense oracle refused: dimension {G.shape[0]} > {DENSE_GUARD}")
    Gd = G.toarray() if hasattr(G, "toarray") else np.asarray(G)
    c = sla.cho_factor(Gd, lower=True)
    return sla.cho_solve(c, np.asarray(b, dtype=np.float64))


def face_spectrum(level: int) -> np.ndarray:
    s = grid.side_of(level)
    t = 2.0 - 2.0 * np.cos(np.pi * np.arange(s) / s)
    return t[:, None] + t[None, :]


def dct_exact(level, A, noise_prec, tau, kappa2, Y, hits=None, prior="laplacian",
              b=None) -> np.ndarray:
    """Exact mu* (component-major vec) via the DCT-II diagonalisation; hits must be 1."""
    if hits is not None and not np.all(np.asarray(hits) == 1.0):
        raise ValueError("dct_exact requires unit hit counts")
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    s = grid.side_of(level)
    if b is None:
        b = model.assemble_rhs(level, A, noise_prec, Y, None)
    Fp = np.asarray(b, dtype=np.float64).reshape(k, s, s)
    Fh = np.stack([dctn(Fp[c], type=2, norm="ortho") for c in range(k)])   # (k, s, s)
    lam = face_spectrum(level)
    lq = kappa2 + (lam if prior == "laplacian" else lam * lam)
    M = A.T @ np.diag(np.asarray(noise_prec, dtype=np.float64)) @ A
    P = np.diag(np.asarray(tau, dtype=np.float64))
    K = M[None, None, :, :] + lq[:, :, None, None] * P[None, None, :, :]   # (s, s, k, k)
    rhs = np.moveaxis(Fh, 0, -1)[..., None]                                 # (s, s, k, 1)
    Xh = np.linalg.solve(K, rhs)[..., 0]                                    # (s, s, k)
    X = np.stack([idctn(Xh[..., c], type=2, norm="ortho") for c in range(k)])
    return X.reshape(-1)


def problem_dct_exact(p) -> np.ndarray:
    return dct_exact(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.Y, p.hits, p.prior)
