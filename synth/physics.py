"""The paper's own workload parameters (App. B; App. C; sec. 4).

Input generation only (no arithmetic of the method): the physical Planck mixing matrix A from the
App. B spectral formulas, the printed noise precisions T, phi_l = 1, and a seeded "paper"
patch -- the paper's simulation protocol (sec. 4 E1: sources iid normal, A and T from App. B,
Y = S A^T + noise per Eq.(model)) on the paper's operator (Q_l = phi_l D^2, kappa2 = 0,
P:L99-106), HEALPix NESTED pixel order inside the face (reading R1) and non-uniform hit counts
N_h (the Planck hit maps are not available: integers 1..4, reading R6 / SURVEY 8(f) NEXT-2).
"""

from __future__ import annotations

import numpy as np

from .problems import PatchProblem

# CODATA 2018 (exact SI values)
H_PLANCK = 6.62607015e-34     # J s
K_BOLTZMANN = 1.380649e-23    # J / K

PLANCK_FREQS_GHZ = (30.0, 44.0, 70.0, 100.0, 143.0, 217.0, 353.0, 545.0, 857.0)
NU0_GHZ = 100.0               # reference frequency: the 4th map
T1_K = 18.1
KAPPA_S = -2.65               # synchrotron spectral index
KAPPA_D = 1.5                 # dust spectral index
KAPPA_FF = -2.14              # free-free
# printed noise precisions T (App. B)
PLANCK_T = (629881.6, 694444.4, 783146.7, 12755102.0, 30864197.5, 30864197.5, 30864197.5, 30864197.5,
            30864197.5)


def _c(nu_hz: np.ndarray) -> np.ndarray:
    """c(nu) = (e^psi - 1)^2 / (psi^2 e^psi), psi = h nu / (k_B T1)."""
    psi = H_PLANCK * nu_hz / (K_BOLTZMANN * T1_K)
    return np.expm1(psi) ** 2 / (psi ** 2 * np.exp(psi))


def _B(nu_hz: np.ndarray) -> np.ndarray:
    """B(nu) = nu / [exp(h nu / k_B T1) - 1]."""
    return nu_hz / np.expm1(H_PLANCK * nu_hz / (K_BOLTZMANN * T1_K))


def planck_mixing(freqs_ghz=PLANCK_FREQS_GHZ, nu0_ghz=NU0_GHZ) -> np.ndarray:
    """n x 4 mixing matrix: CMB (ones), synchrotron, dust, free-free (App. B)."""
    nu = np.asarray(freqs_ghz, dtype=np.float64) * 1e9
    nu0 = nu0_ghz * 1e9
    r = nu / nu0
    c = _c(nu)
    A = np.empty((nu.size, 4))
    A[:, 0] = 1.0
    A[:, 1] = c * r ** KAPPA_S
    A[:, 2] = c * _B(nu) / _B(np.array([nu0]))[0] * r ** KAPPA_D
    A[:, 3] = c * r ** KAPPA_FF
    return A


def nested_order(maps: np.ndarray) -> np.ndarray:
    """[..][side][side] row-major maps -> the same maps with pixels in HEALPix NESTED order inside the
    face (reading R1: bit b of x -> bit 2b, bit b of y -> bit 2b+1 of the index), reshaped back to
    [..][side][side] -- how the paper's HEALPix data arrive (App. A)."""
    maps = np.asarray(maps)
    side = maps.shape[-1]
    y, x = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    idx = np.zeros((side, side), dtype=np.int64)
    for b in range(max(1, int(side).bit_length())):
        idx |= ((x >> b) & 1) << (2 * b)
        idx |= ((y >> b) & 1) << (2 * b + 1)
    flat = maps.reshape(maps.shape[:-2] + (side * side,))
    out = np.empty_like(flat)
    out[..., idx.reshape(-1)] = flat
    return out.reshape(maps.shape)


def make_paper_patch(level: int, seed: int, hits="random", kappa2: float = 0.0) -> PatchProblem:
    """One face of the paper's simulation (sec. 4) in HEALPix NESTED order is produced by
    the caller permuting Y / hits; this returns the row-major maps.  Draw order with
    rng = Generator(PCG64(seed)): 1. S ~ N(0, 1) iid [m][side][side]; 2. noise E ~ N(0, 1/T) [N][n];
    3. hits integers 1..4 [side][side] (if hits == "random")."""
    side = 1 << level
    N = side * side
    A = planck_mixing()
    n, k = A.shape
    T = np.asarray(PLANCK_T, dtype=np.float64)
    rng = np.random.Generator(np.random.PCG64(seed))
    S = rng.standard_normal((k, side, side))
    E = rng.standard_normal((N, n)) / np.sqrt(T)[None, :]
    Y = np.ascontiguousarray((S.reshape(k, N).T @ A.T + E).T.reshape(n, side, side))
    h = rng.integers(1, 5, size=(side, side)).astype(np.float64) if hits == "random" else None
    return PatchProblem(level=level, A=A, noise_prec=T, tau=np.ones(k), kappa2=float(kappa2), Y=Y, S=S,
                        hits=h, prior="d2", seed=seed, meta={"workload": "paper (App. B physics)"})
