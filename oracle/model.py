"""Oracle: literal Kronecker assembly of the posterior system (Q + B^T C B) mu = B^T C Y.

PAPER.md:
  * Sec. 2.1 P:L49-53 -- curly-Y stacked by map, B = A (x) I_N, C diagonal precision.
  * Sec. 3 P:L107-112 -- C = diag(tau_1..tau_n) (x) diag(n_1..n_N) = T (x) N (hit counts).
  * Sec. 3.1 P:L140-148 -- Q = P (x) D^2, P = diag(phi_l) (per-source prior scale).
  * Eq.(Q*) P:L73-77, Eq.(mu*) P:L78-82, Eq.(Axb) P:L95-98 -- G = Q + B^T C B, b = B^T C Y.
Readings: R3/R24 the prior block of component l is phi_l * Q0 with
Q0 = kappa2 I + L ("laplacian", BASELINE configs) or Q0 = D^2 + kappa2 I ("d2", the
paper's phi D^2); R5 the configs' tau_i are the paper's phi_l; R6 T = 1/sigma^2.

Vectors are the paper's vec(): component-major stacking, mu[l*N + j] = source l at
pixel j.  Everything is assembled with scipy.sparse -- nothing
matrix-free, no fusion.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import grid


def prior_Q0(level: int, kappa2: float, prior: str = "laplacian", layout: str = "row") -> sp.csr_matrix:
    """Single-source prior precision Q0 (before the per-source scale phi_l), pixels in `layout`."""
    N = grid.side_of(level) ** 2
    I = sp.identity(N, format="csr")
    if prior == "laplacian":
        return (kappa2 * I + grid.laplacian(level, layout)).tocsr()
    if prior == "d2":
        D = grid.D_matrix(level, layout)
        return (D @ D + kappa2 * I).tocsr()
    raise ValueError(f"unknown prior {prior!r}")


def _hits_vec(level: int, hits) -> np.ndarray:
    N = grid.side_of(level) ** 2
    if hits is None:
        return np.ones(N)
    h = np.asarray(hits, dtype=np.float64).reshape(N)
    return h


def B_matrix(level: int, A: np.ndarray) -> sp.csr_matrix:
    """B = A (x) I_N."""
    N = grid.side_of(level) ** 2
    return sp.kron(sp.csr_matrix(np.asarray(A, dtype=np.float64)),
                   sp.identity(N, format="csr"), format="csr")


def C_matrix(level: int, noise_prec: np.ndarray, hits=None) -> sp.csr_matrix:
    """C = T (x) N_h, diagonal."""
    h = _hits_vec(level, hits)
    return sp.diags(np.kron(np.asarray(noise_prec, dtype=np.float64), h)).tocsr()


def Q_matrix(level: int, tau: np.ndarray, kappa2: float, prior: str = "laplacian",
             layout: str = "row") -> sp.csr_matrix:
    """Q = P (x) Q0, P = diag(phi)."""
    return sp.kron(sp.diags(np.asarray(tau, dtype=np.float64)),
                   prior_Q0(level, kappa2, prior, layout), format="csr")


def assemble_G(level, A, noise_prec, tau, kappa2, hits=None, prior="laplacian", layout="row") -> sp.csr_matrix:
    """G = Q + B^T C B  (Eq.(Q*) P:L75, Eq.(Axb)), literal sparse assembly.  `hits` is a
    vector in the same pixel layout as the grid."""
    B = B_matrix(level, A)
    C = C_matrix(level, noise_prec, hits)
    Q = Q_matrix(level, tau, kappa2, prior, layout)
    return (B.T @ C @ B + Q).tocsr()


def vec_maps(Y: np.ndarray) -> np.ndarray:
    """curly-Y = (Y_1, ..., Y_n) stacked by map."""
    Y = np.asarray(Y, dtype=np.float64)
    return Y.reshape(Y.shape[0], -1).reshape(-1)


def assemble_rhs(level, A, noise_prec, Y, hits=None) -> np.ndarray:
    """b = B^T C curly-Y  (Eq.(mu*) P:L80)."""
    B = B_matrix(level, A)
    C = C_matrix(level, noise_prec, hits)
    return B.T @ (C @ vec_maps(Y))


def to_layout(level: int, maps: np.ndarray, layout: str) -> np.ndarray:
    """Maps stored as [..][side][side] (row, column) -> [..][N] vectors in `layout` order."""
    maps = np.asarray(maps, dtype=np.float64)
    s = grid.side_of(level)
    flat = maps.reshape(maps.shape[:-2] + (s * s,))
    if layout == "row":
        return flat.copy()
    out = np.empty_like(flat)
    out[..., grid.pixel_index(level, layout).reshape(-1)] = flat
    return out


def problem_system(p, layout: str = "row"):
    """(G, b) for a synth.PatchProblem-like object, pixels numbered in `layout`."""
    hits = None if p.hits is None else to_layout(p.level, p.hits, layout)
    G = assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2, hits, p.prior, layout)
    b = assemble_rhs(p.level, p.A, p.noise_prec, to_layout(p.level, p.Y, layout), hits)
    return G, b


def apply_G_rows(level, A, noise_prec, tau, kappa2, x, rows, hits=None, prior="laplacian"):
    """(G x) at selected rows, one at a time, from the posterior's summation form.

    Row (l, j) of G x is, by Eq.(Q*) written entrywise (likelihood Eq.(2) P:L54-57 and
    prior Eq.(3) P:L62-65 with Q = P (x) Q0):
        sum_f A_fl T_f h_j sum_d A_fd x_{d,j}  +  phi_l (Q0 x_l)_j
    with (L v)_j = sum_{j' in nbrs(j)} (v_j - v_j')  and  D = -L.
    ``x`` is (k, N); ``rows`` is a list of (l, j).  Used for sampled full-size parity.
    """
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    x = np.asarray(x, dtype=np.float64).reshape(k, -1)
    h = _hits_vec(level, hits)
    out = []

    def Lv(v, j):
        nb = grid.neighbors(level, j)
        return sum(v[j] - v[i] for i in nb)

    for (l, j) in rows:
        lik = 0.0
        for f in range(n):
            s = 0.0
            for d in range(k):
                s += A[f, d] * x[d, j]
            lik += A[f, l] * noise_prec[f] * h[j] * s
        if prior == "laplacian":
            pr = kappa2 * x[l, j] + Lv(x[l], j)
        else:  # D^2 + kappa2 I, (D^2 v)_j = sum_i D_ji (D v)_i, D = -L
            nb = grid.neighbors(level, j)
            Dv_j = -Lv(x[l], j)
            acc = -len(nb) * Dv_j
            for i in nb:
                acc += -Lv(x[l], i)
            pr = acc + kappa2 * x[l, j]
        out.append(lik + tau[l] * pr)
    return np.array(out)


def neg_log_posterior(level, A, noise_prec, tau, kappa2, Y, S, hits=None, prior="laplacian"):
    """-log p(S | Y) up to a constant, written from Eq.(2) and Eq.(3) entrywise.

    1/2 sum_j sum_f T_f h_j (y_jf - sum_l A_fl s_jl)^2 + 1/2 sum_l phi_l s_l^T Q0 s_l.
    Its Hessian is G and its gradient at S = 0 is -b (Eq.(Q*), Eq.(mu*)); used as a pin.
    The prior quadratic form is written as edge differences: s^T L s = sum_edges (s_i - s_j)^2.
    """
    A = np.asarray(A, dtype=np.float64)
    n, k = A.shape
    s_side = grid.side_of(level)
    N = s_side * s_side
    S = np.asarray(S, dtype=np.float64).reshape(k, N)
    Yf = np.asarray(Y, dtype=np.float64).reshape(n, N)
    h = _hits_vec(level, hits)
    val = 0.0
    for j in range(N):
        for f in range(n):
            pred = sum(A[f, l] * S[l, j] for l in range(k))
            val += 0.5 * noise_prec[f] * h[j] * (Yf[f, j] - pred) ** 2
    for l in range(k):
        s = S[l]
        if prior == "laplacian":
            q = kappa2 * float(s @ s)
            for j in range(N):
                for i in grid.neighbors(level, j):
                    if i > j:
                        q += (s[j] - s[i]) ** 2
        else:
            Ds = np.array([sum(s[i] for i in grid.neighbors(level, j)) -
                           len(grid.neighbors(level, j)) * s[j] for j in range(N)])
            q = float(Ds @ Ds) + kappa2 * float(s @ s)
        val += 0.5 * tau[l] * q
    return val
