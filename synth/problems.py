"""Seeded problem generator (SURVEY.md section 8(d) recipe; BASELINE.json `configs`).

Per patch, with ``rng = numpy.random.Generator(numpy.random.PCG64(seed))``,
draws in this exact order:

1. ``A = rng.uniform(0.1, 2.0, (n, k)); A[:, 0] = 1``    (CMB column of ones)
2. ``sigma2 = exp(rng.uniform(log 1e-2, 0, n))``; noise precision ``T = 1/sigma2``
   (paper's C = T (x) N_h; config "noise variances LogUniform(1e-2,1)")
3. per-component prior scales tau (paper's phi_l, matrix P):
   ``fixed3`` -> [1, 10, 100] (tiny/medium); ``loguniform`` -> exp(U(0, log 1e3)) per
   component (planck/fullsky); ``logspace`` -> logspace(0, 4, k) (stress, no draw)
4. kappa2: 0.1 (no draw), or ``exp(rng.uniform(log 1e-3, 0))`` (stress)
5. sources: for each component i, ``z = rng.standard_normal((side, side))`` and
   ``s_i = idctn(z / sqrt(tau_i * lam), type=2, norm='ortho')`` -- an exact draw from the
   Gaussian prior with precision tau_i * Q0 (lam is the spectrum of Q0 on the free-boundary
   face grid; a sampling device for the inputs only).
6. ``E = rng.standard_normal((N, n)) * sqrt(sigma2)``
7. ``Y = S A^T + E`` (PAPER.md Eq.(model)), stored as planes ``[n][side][side]``.

Hit counts are all ones unless a test asks for random ones (``hits="random"`` draws
integers 1..4 *after* step 7 so the other arrays are unchanged).

Nothing here computes the operator, the right-hand side or any solver step.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy.fft import idctn

# BASELINE.json "configs" (in order): tiny, medium, planck, fullsky, stress.
CONFIGS = {
    "tiny": dict(level=5, n=9, k=3, seeds=[0], tau="fixed3", kappa2="fixed"),
    "medium": dict(level=8, n=9, k=3, seeds=[1], tau="fixed3", kappa2="fixed"),
    "planck": dict(level=10, n=9, k=4, seeds=[2], tau="loguniform", kappa2="fixed"),
    "fullsky": dict(level=10, n=9, k=4, seeds=list(range(100, 112)), tau="loguniform",
                    kappa2="fixed"),
    "stress": dict(level=11, n=9, k=6, seeds=[3], tau="logspace", kappa2="loguniform"),
}


@dataclass
class PatchProblem:
    """One base patch (face) of the source-separation problem."""

    level: int
    A: np.ndarray            # (n, k) mixing matrix
    noise_prec: np.ndarray   # (n,) T = 1/sigma^2
    tau: np.ndarray          # (k,) per-component prior scales (paper phi, matrix P)
    kappa2: float            # prior nugget
    Y: np.ndarray            # (n, side, side) data maps
    S: np.ndarray            # (k, side, side) true sources
    hits: Optional[np.ndarray] = None   # (side, side) hit counts or None (= ones)
    prior: str = "laplacian"
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def side(self) -> int:
        return 1 << self.level

    @property
    def N(self) -> int:
        return self.side * self.side

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def k(self) -> int:
        return self.A.shape[1]


def _grid_spectrum(side: int, prior: str, kappa2: float) -> np.ndarray:
    """Spectrum of the prior precision on the face grid, used only to draw the sources."""
    t = 2.0 - 2.0 * np.cos(np.pi * np.arange(side) / side)
    lam = t[:, None] + t[None, :]
    if prior == "laplacian":
        return kappa2 + lam
    if prior == "d2":
        return kappa2 + lam * lam
    raise ValueError(f"unknown prior {prior!r}")


def make_patch(level: int, n: int, k: int, seed: int, tau: str = "fixed3",
               kappa2="fixed", prior: str = "laplacian", hits=None,
               tau_values=None, kappa2_value=None) -> PatchProblem:
    """Draw one patch with the section-8(d) recipe.

    ``tau``: "fixed3" | "loguniform" | "logspace" | "given" (then ``tau_values``).
    ``kappa2``: "fixed" (0.1) | "loguniform" | "given" (then ``kappa2_value``).
    ``hits``: None | "random" | array (side, side).
    """
    if level < 0 or level > 12:
        raise ValueError("level must be in [0, 12]")
    side = 1 << level
    N = side * side
    rng = np.random.Generator(np.random.PCG64(seed))
    # 1. mixing matrix
    A = rng.uniform(0.1, 2.0, (n, k))
    A[:, 0] = 1.0
    # 2. noise variances -> precisions
    sigma2 = np.exp(rng.uniform(np.log(1e-2), 0.0, n))
    noise_prec = 1.0 / sigma2
    # 3. prior scales
    if tau == "fixed3":
        base = np.array([1.0, 10.0, 100.0])
        tau_v = np.resize(base, k).astype(np.float64)
    elif tau == "loguniform":
        tau_v = np.exp(rng.uniform(0.0, np.log(1e3), k))
    elif tau == "logspace":
        tau_v = np.logspace(0.0, 4.0, k)
    elif tau == "given":
        tau_v = np.asarray(tau_values, dtype=np.float64).copy()
        assert tau_v.shape == (k,)
    else:
        raise ValueError(tau)
    # 4. nugget
    if kappa2 == "fixed":
        k2 = 0.1
    elif kappa2 == "loguniform":
        k2 = float(np.exp(rng.uniform(np.log(1e-3), 0.0)))
    elif kappa2 == "given":
        k2 = float(kappa2_value)
    else:
        raise ValueError(kappa2)
    # 5. sources from the prior
    lam = _grid_spectrum(side, prior, k2)
    S = np.empty((k, side, side))
    for i in range(k):
        z = rng.standard_normal((side, side))
        with np.errstate(divide="ignore", invalid="ignore"):
            scale = np.where(lam > 0, 1.0 / np.sqrt(tau_v[i] * np.where(lam > 0, lam, 1.0)), 0.0)
        S[i] = idctn(z * scale, type=2, norm="ortho")
    # 6. noise
    E = rng.standard_normal((N, n)) * np.sqrt(sigma2)[None, :]
    # 7. data
    Yflat = S.reshape(k, N).T @ A.T + E          # (N, n)
    Y = np.ascontiguousarray(Yflat.T.reshape(n, side, side))
    h = None
    if isinstance(hits, str) and hits == "random":
        h = rng.integers(1, 5, size=(side, side)).astype(np.float64)
    elif hits is not None:
        h = np.asarray(hits, dtype=np.float64).reshape(side, side)
    return PatchProblem(level=level, A=A, noise_prec=noise_prec, tau=tau_v, kappa2=k2,
                        Y=Y, S=S, hits=h, prior=prior, seed=seed)


def make_config(name: str, patches: Optional[list] = None, prior: str = "laplacian"):
    """All patches of a named BASELINE config (optionally a subset of patch indices)."""
    c = CONFIGS[name]
    seeds = c["seeds"]
    idx = range(len(seeds)) if patches is None else patches
    return [make_patch(c["level"], c["n"], c["k"], seeds[i], tau=c["tau"],
                       kappa2=c["kappa2"], prior=prior) for i in idx]


def config_patches(name: str) -> int:
    return len(CONFIGS[name]["seeds"])


def stack(problems):
    """Stack a list of patches into the C-ABI host layouts (all patches same shape).

    Returns dict with A [P][n][k], noise_prec [P][n], tau [P][k], kappa2 [P],
    Y [P][n][side][side], hits [P][side][side] or None.
    """
    A = np.ascontiguousarray(np.stack([p.A for p in problems]))
    T = np.ascontiguousarray(np.stack([p.noise_prec for p in problems]))
    tau = np.ascontiguousarray(np.stack([p.tau for p in problems]))
    k2 = np.array([p.kappa2 for p in problems], dtype=np.float64)
    Y = np.ascontiguousarray(np.stack([p.Y for p in problems]))
    if any(p.hits is not None for p in problems):
        hits = np.ascontiguousarray(np.stack([
            p.hits if p.hits is not None else np.ones((p.side, p.side)) for p in problems]))
    else:
        hits = None
    return dict(A=A, noise_prec=T, tau=tau, kappa2=k2, Y=Y, hits=hits)
