"""Pins for oracle.sylvester: Lemma 2, the Kronecker/Sylvester identity, exact solutions."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import exact, grid, model, sylvester
from synth import make_config, make_patch


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_lemma2_and_eigen_normalisation():
    p = make_patch(2, 9, 4, seed=5, tau="loguniform")
    M, P, rho, W = sylvester.small_factor(p.A, p.noise_prec, p.tau)
    Shat = M @ np.linalg.inv(P)                       # S^ = A^T T A P^{-1}
    Pinv = np.linalg.inv(P)
    # Lemma 2: P^{-1} S^ = S^T P^{-1}
    assert np.abs(Pinv @ Shat - Shat.T @ Pinv).max() <= 1e-12 * np.abs(Pinv @ Shat).max()
    assert np.allclose(W.T @ P @ W, np.eye(4), atol=1e-12)
    assert np.allclose(M @ W, P @ W @ np.diag(rho), atol=1e-9 * np.abs(M).max())
    assert np.all(np.diff(rho) >= 0) and rho.min() > 0
    U = P @ W                                          # paper's U: S^ = U R U^{-1}, U^T P^{-1} U = I
    assert np.allclose(U.T @ Pinv @ U, np.eye(4), atol=1e-12)
    assert np.allclose(Shat @ U, U @ np.diag(rho), atol=1e-9 * np.abs(Shat).max())
    for i in range(4):
        assert W[np.argmax(np.abs(W[:, i])), i] > 0


@pytest.mark.parametrize("hits", [None, "random"])
def test_kronecker_sylvester_identity(hits):
    # north star: vec(Q0 X P + N_h X M) = (P (x) Q0 + M (x) N_h) vec X = G vec X
    p = make_patch(3, 9, 4, seed=8, tau="loguniform", hits=hits)
    G = model.assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits)
    Q0 = model.prior_Q0(p.level, p.kappa2)
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    Nh = sp.diags(np.ones(p.N) if p.hits is None else p.hits.ravel())
    X = np.random.default_rng(0).standard_normal((p.N, 4))
    lhs = (Q0 @ X) @ np.diag(p.tau) + (Nh @ X) @ M
    y = G @ X.T.reshape(-1)
    assert np.abs(lhs.T.reshape(-1) - y).max() <= 5e-16 * 50 * np.abs(y).max()


def test_sylvester_tiny_matches_exact():
    p = make_config("tiny")[0]
    res = sylvester.problem_solve(p, tol=1e-10)
    G, b = model.problem_system(p)
    x_star = exact.dense_solve(G, b)
    assert res.converged
    assert rel(res.x, x_star) <= 1e-8
    assert rel(res.x, exact.problem_dct_exact(p)) <= 1e-8
    assert len(res.iterations) == 3 and all(i > 0 for i in res.iterations)


def test_sylvester_with_hits_matches_dense():
    p = make_patch(4, 9, 3, seed=12, hits="random")
    res = sylvester.problem_solve(p, tol=1e-11)
    G, b = model.problem_system(p)
    assert rel(res.x, exact.dense_solve(G, b)) <= 1e-8


def test_sylvester_k1_is_single_shifted_system():
    p = make_patch(3, 4, 1, seed=1, tau="given", tau_values=[3.0])
    M, P, rho, W = sylvester.small_factor(p.A, p.noise_prec, p.tau)
    m = float(p.A[:, 0] @ (p.noise_prec * p.A[:, 0]))
    assert np.isclose(rho[0], m / 3.0) and np.isclose(W[0, 0], 1 / np.sqrt(3.0))
    res = sylvester.problem_solve(p)
    G, b = model.problem_system(p)
    assert rel(res.x, exact.dense_solve(G, b)) <= 1e-8


def test_sylvester_jacobi_preconditioned():
    """The Jacobi option (diag of the shifted operator) changes the iterates, not the solution."""
    p = make_patch(4, 9, 3, seed=12, hits="random")
    plain = sylvester.problem_solve(p, tol=1e-11)
    pc = sylvester.problem_solve(p, tol=1e-11, precond="jacobi")
    G, b = model.problem_system(p)
    x_star = exact.dense_solve(G, b)
    assert pc.converged and rel(pc.x, x_star) <= 1e-8
    assert pc.iterations != plain.iterations


@pytest.mark.slow
def test_sylvester_medium_matches_dct():
    p = make_config("medium")[0]
    res = sylvester.problem_solve(p, tol=1e-10)
    assert rel(res.x, exact.problem_dct_exact(p)) <= 1e-8


# ----------------------------------------------------------------------- block-Lanczos (NEXT-1)
def test_lanczos_tiny_medium_match_exact():
    from oracle import lanczos
    for name in ("tiny", "medium"):
        p = make_config(name)[0]
        r = lanczos.problem_solve(p, tol=1e-10)
        assert r.converged
        assert rel(r.x, exact.problem_dct_exact(p)) <= 1e-8


def test_lanczos_relation_orthonormality_and_galerkin():
    """Early steps (orthogonality intact): AA V_j = V_{j+1} T_j (Lanczos relation), V^T N V = I,
    and the Galerkin solution satisfies T Z + Z S^ = E_1 B_0 (Eq.(Sylv-small))."""
    from oracle import grid, lanczos, model as mdl
    p = make_patch(4, 9, 3, seed=21, tau="loguniform", hits="random")
    r = lanczos.problem_solve(p, tol=1e-30, max_iter=4, keep_basis=True)
    m, h = p.k, p.hits.reshape(-1)
    Vs = np.hstack(r.V)                                   # N x 4m
    assert np.abs(Vs.T @ (h[:, None] * Vs) - np.eye(4 * m)).max() <= 1e-10
    Q0 = mdl.prior_Q0(p.level, p.kappa2)
    AV = (Q0 @ Vs[:, :3 * m]) / h[:, None]
    T = np.zeros((4 * m, 3 * m))
    for a in range(3):
        T[a * m:(a + 1) * m, a * m:(a + 1) * m] = r.H[a]
        T[(a + 1) * m:(a + 2) * m, a * m:(a + 1) * m] = r.B[a + 1]
        if a + 1 < 3:
            T[a * m:(a + 1) * m, (a + 1) * m:(a + 2) * m] = r.B[a + 1].T
    assert np.abs(AV - Vs @ T).max() <= 1e-9 * np.abs(AV).max()


def test_lanczos_residual_estimate_is_the_u_basis_residual():
    """Paper's gamma (reading R26) = ||(AA M + M S^ - Y^) U||_N,F^2 for the Galerkin
    iterate M_j = V Z (checked while the basis is still orthonormal)."""
    from oracle import lanczos, model as mdl
    from oracle.sylvester import small_factor
    p = make_patch(4, 9, 3, seed=22, tau="loguniform")
    for steps in (2, 4):
        r = lanczos.problem_solve(p, tol=1e-30, max_iter=steps, keep_basis=True)
        m, N = p.k, p.N
        Mk, P, rho, W = small_factor(p.A, p.noise_prec, p.tau)
        U = P @ W
        Yhat = (p.Y.reshape(p.n, N).T @ np.diag(p.noise_prec) @ p.A) @ np.linalg.inv(P)
        M = r.x.reshape(m, N).T
        Q0 = mdl.prior_Q0(p.level, p.kappa2)
        R = Q0 @ M + M @ (Mk @ np.linalg.inv(P)) - Yhat
        est = r.gamma_history[-1] * np.linalg.norm(r.B[0])
        assert np.isclose(np.linalg.norm(R @ U), est, rtol=1e-6), (np.linalg.norm(R @ U), est)


def test_lanczos_k1_is_plain_lanczos_on_the_shifted_system():
    """m = 1: S^ = rho (scalar); the solution of (N^{-1} Q0 + rho) x = y^ (dense solve)."""
    from oracle import lanczos
    p = make_patch(3, 4, 1, seed=1, tau="given", tau_values=[2.0])
    r = lanczos.problem_solve(p, tol=1e-12)
    G, b = model.problem_system(p)
    assert rel(r.x, exact.dense_solve(G, b)) <= 1e-9


@pytest.mark.parametrize("level,seed", [(5, 70), (6, 70)])
def test_lanczos_with_hits_matches_the_direct_solve(level, seed):
    """Non-uniform hits: N_h^{-1} Q0 is only N-symmetric (Lemma 1) and the basis loses
    orthogonality early (max |V^T N V - I| ~ 0.2 at L = 6).  The second Lanczos pass must then
    rebuild the first pass's blocks exactly (Alg. SylvSolver, reading R30): a replay
    whose V_1 = Y^ B_0^{-1} is rounded differently from the first pass's drifts to ~1e-6."""
    import scipy.sparse.linalg as ssl
    from oracle import lanczos
    p = make_patch(level, 9, 3, seed=seed, tau="loguniform", hits="random")
    r = lanczos.problem_solve(p, tol=1e-10)
    G, b = model.problem_system(p)
    ref = ssl.spsolve(G.tocsc(), b)
    assert r.converged
    assert rel(r.x, ref) <= 5e-9
