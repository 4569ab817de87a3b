"""Pins for oracle.kohler (Alg. Kohler, reading R33)."""

import numpy as np
import scipy.sparse.linalg as ssl

from oracle import exact, kohler, model
from synth import make_config, make_patch


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_canonical_schur_factor():
    p = make_patch(2, 9, 5, seed=31, tau="loguniform")
    S, W, R = kohler.schur_factor(p.A, p.noise_prec, p.tau)
    assert np.allclose(W.T @ W, np.eye(5), atol=1e-13)                       # orthogonal
    assert np.allclose(W @ R @ W.T, S, atol=1e-10 * np.abs(S).max())         # S = W R W^T
    assert np.abs(np.tril(R, -1)).max() <= 1e-10 * np.abs(R).max()          # upper triangular
    ev = np.sort(np.linalg.eigvals(S).real)
    assert np.allclose(np.diag(R), ev, rtol=1e-10)                           # ascending eigenvalues
    assert np.any(np.abs(np.triu(R, 1)) > 1e-6 * np.abs(R).max())            # genuinely non-normal


def test_kohler_matches_exact_solutions():
    for name in ("tiny", "medium"):
        p = make_config(name)[0]
        r = kohler.problem_solve(p, tol=1e-10)
        assert r.converged
        assert rel(r.x, exact.problem_dct_exact(p)) <= 1e-8


def test_kohler_with_hits_and_d2_matches_the_direct_solve():
    for prior in ("laplacian", "d2"):
        p = make_patch(4, 9, 4, seed=32, tau="loguniform", hits="random", prior=prior)
        r = kohler.problem_solve(p, tol=1e-12)
        G, b = model.problem_system(p)
        assert rel(r.x, ssl.spsolve(G.tocsc(), b)) <= 1e-8


def test_kohler_k1_is_one_shifted_solve():
    p = make_patch(3, 4, 1, seed=33, tau="given", tau_values=[3.0])
    r = kohler.problem_solve(p, tol=1e-12)
    G, b = model.problem_system(p)
    assert rel(r.x, exact.dense_solve(G, b)) <= 1e-9
    assert r.W.shape == (1, 1) and abs(abs(r.W[0, 0]) - 1.0) < 1e-15
