"""Oracle: posterior variances diag(Q^-1) ("of most importance ... the main
diagonal") -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper computes the posterior mean only; for the variances it names the target, not a method.
The build uses Hutchinson's estimator (reading R32): with Rademacher probes z_i (entries +-1),
    diag(G^{-1}) ~= (1/s) sum_i z_i (.) G^{-1} z_i,
unbiased because E[z z^T] = I, with Var = (1/s) sum_{l != j} (G^{-1})_{jl}^2 per entry.  The probes
come from a counter-based generator that the GPU path implements independently (the C ABI header
documents it): z_i[p][c][j] = sign bit of splitmix64(splitmix64(seed) + ((i P + p) k + c) N + j)
(1 -> -1, 0 -> +1), SplitMix64 = Steele, Lea & Flood (2014) with Vigna's constants.  Each probe is
solved with the oracle's textbook CG (oracle.cg.cg_hs).  exact_diag is the direct reference.
"""

from __future__ import annotations

import numpy as np

from . import cg

_M64 = (1 << 64) - 1


def splitmix64(x):
    """SplitMix64 output for state x (Python ints or numpy uint64 arrays, arithmetic mod 2^64)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def rademacher(seed: int, probe: int, P: int, k: int, N: int) -> np.ndarray:
    """Probe `probe` for P patches: array [P][k][N] of +-1 (pixel index j in the system's numbering)."""
    s0 = splitmix64(np.uint64(seed & _M64))
    key = (np.uint64(probe) * np.uint64(P * k) + np.arange(P * k, dtype=np.uint64)[:, None]) * np.uint64(N) \
        + np.arange(N, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        bits = splitmix64(s0 + key) >> np.uint64(63)
    return np.where(bits == 1, -1.0, 1.0).reshape(P, k, N)


def hutchinson(systems, k: int, N: int, n_probes: int, seed: int, tol: float = 1e-10, solve=None) -> np.ndarray:
    """systems: P assembled G (k N x k N, component-major vec).  Returns var [P][k N].
    solve(G, z) defaults to the oracle CG to `tol`; pass an exact solver for statistical pins."""
    P = len(systems)
    acc = np.zeros((P, k * N))
    for i in range(n_probes):
        Z = rademacher(seed, i, P, k, N).reshape(P, k * N)
        for p, G in enumerate(systems):
            x = solve(G, Z[p]) if solve is not None else cg.cg_hs(G, Z[p], tol=tol, max_iter=100000).x
            acc[p] += Z[p] * x
    return acc / n_probes


def exact_diag(G) -> np.ndarray:
    """diag(G^{-1}) by a dense inverse (small systems only)."""
    Gd = G.toarray() if hasattr(G, "toarray") else np.asarray(G)
    return np.diag(np.linalg.inv(Gd)).copy()


def dct_diag_moments(level: int, A, noise_prec, tau, kappa2, prior: str = "laplacian"):
    """hits = 1: (diag(G^-1), diag(G^-2)) [k][N] in closed form.  G = sum_ab (v_ab v_ab^T) (x) K_ab with
    the orthonormal 2-D DCT-II modes v_ab(y, x) = u_a(y) u_b(x) and K_ab = M + lam^{Q0}_ab P (the
    diagonalisation of oracle.exact.dct_exact), so
        diag(G^-p)[c](y, x) = sum_a u_a(y)^2 sum_b u_b(x)^2 [K_ab^-p]_cc,   p = 1, 2,
    evaluated as two matrix products per component.  diag(G^-2)_j = sum_l (G^-1)_jl^2 gives the
    Hutchinson standard error at any size."""
    A = np.asarray(A, dtype=np.float64)
    k = A.shape[1]
    s = 1 << level
    t = 2.0 - 2.0 * np.cos(np.pi * np.arange(s) / s)
    lam = t[:, None] + t[None, :]
    lq = kappa2 + (lam if prior == "laplacian" else lam * lam)
    M = A.T @ np.diag(np.asarray(noise_prec, dtype=np.float64)) @ A
    P = np.diag(np.asarray(tau, dtype=np.float64))
    Kab = M[None, None] + lq[:, :, None, None] * P[None, None]                 # (s, s, k, k)
    Ki = np.linalg.inv(Kab)
    Ki2 = Ki @ Ki
    u = np.sqrt(2.0 / s) * np.cos(np.pi * np.outer(np.arange(s) + 0.5, np.arange(s)) / s)
    u[:, 0] = np.sqrt(1.0 / s)
    u2 = u ** 2                                                                 # [y, a]
    d1 = np.stack([u2 @ Ki[:, :, c, c] @ u2.T for c in range(k)]).reshape(k, s * s)
    d2 = np.stack([u2 @ Ki2[:, :, c, c] @ u2.T for c in range(k)]).reshape(k, s * s)
    return d1, d2
