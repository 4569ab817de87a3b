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
