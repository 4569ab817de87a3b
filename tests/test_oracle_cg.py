"""Pins for oracle.cg and oracle.exact: exact solves, library CG, textbook CG invariants."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import cg, exact, model
from synth import make_config, make_patch


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def tiny():
    p = make_config("tiny")[0]
    G, b = model.problem_system(p)
    return p, G, b


def test_dct_exact_equals_dense_cholesky(tiny):
    p, G, b = tiny
    x_dense = exact.dense_solve(G, b)
    x_dct = exact.problem_dct_exact(p)
    assert rel(x_dct, x_dense) <= 1e-12
    assert np.linalg.norm(G @ x_dense - b) <= 1e-12 * np.linalg.norm(b)


def test_dense_guard():
    p = make_patch(6, 9, 3, seed=0)
    G, b = model.problem_system(p)
    with pytest.raises(MemoryError):
        exact.dense_solve(G, b)


def test_cg_tiny_matches_exact_and_scipy(tiny):
    p, G, b = tiny
    res = cg.cg_hs(G, b, tol=1e-10)
    assert res.converged
    x_star = exact.dense_solve(G, b)
    assert rel(res.x, x_star) <= 1e-8
    assert np.linalg.norm(b - G @ res.x) <= 1.01e-10 * np.linalg.norm(b) * 1.5
    # scipy's CG is an independent implementation of the same textbook iteration
    its = []
    x_sp, info = spla.cg(G, b, rtol=1e-10, atol=0.0, maxiter=10000,
                         callback=lambda xk: its.append(1))
    assert info == 0
    assert abs(len(its) - res.iterations) <= 1
    assert rel(res.x, x_sp) <= 1e-9
    assert len(res.history) == res.iterations
    assert res.history[-1] <= 1e-10 < res.history[-2]


def test_cg_zero_rhs():
    p = make_patch(3, 9, 3, seed=0)
    G, b = model.problem_system(p)
    res = cg.cg_hs(G, np.zeros_like(b))
    assert res.iterations == 0 and res.converged and not res.x.any()
    res2 = cg.cg_single_pass(G, np.zeros_like(b))
    assert res2.iterations == 0 and res2.converged


def test_finite_termination_level1():
    # mN = 8: CG terminates in at most mN iterations
    p = make_patch(1, 3, 2, seed=2, tau="given", tau_values=[1.0, 3.0])
    G, b = model.problem_system(p)
    res = cg.cg_hs(G, b, tol=1e-12)
    assert res.converged and res.iterations <= 8


def test_energy_norm_monotone_and_orthogonality():
    p = make_patch(2, 9, 3, seed=4)
    G, b = model.problem_system(p)
    x_star = exact.dense_solve(G, b)
    errs, rs = [], []

    def cb(j, x, r):
        e = x - x_star
        errs.append(float(e @ (G @ e)))
        rs.append(r.copy())

    cg.cg_hs(G, b, tol=1e-14, max_iter=200, callback=cb)
    e0 = float(x_star @ (G @ x_star))
    seq = [e0] + errs
    assert all(seq[i + 1] <= seq[i] * (1 + 1e-12) + 1e-300 for i in range(len(seq) - 1))
    R = [b] + rs[:10]
    for i in range(len(R)):
        for j in range(i):
            c = abs(R[i] @ R[j]) / (np.linalg.norm(R[i]) * np.linalg.norm(R[j]))
            assert c <= 1e-8


def test_linearity(tiny):
    p, G, b = tiny
    r1 = cg.cg_hs(G, b, tol=1e-10)
    r2 = cg.cg_hs(G, 3.5 * b, tol=1e-10)
    assert r1.iterations == r2.iterations
    assert rel(r2.x, 3.5 * r1.x) <= 1e-12


def test_single_pass_variant_like_hs(tiny):
    p, G, b = tiny
    hs = cg.cg_hs(G, b, tol=1e-10)
    sp1 = cg.cg_single_pass(G, b, tol=1e-10)
    assert sp1.converged and abs(sp1.iterations - hs.iterations) <= 1
    assert rel(sp1.x, hs.x) <= 1e-10


def test_block_jacobi_precond(tiny):
    p, G, b = tiny
    K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2)
    hs = cg.cg_hs(G, b, tol=1e-10)
    pc = cg.cg_hs(G, b, tol=1e-10, precond=K)
    sp1 = cg.cg_single_pass(G, b, tol=1e-10, precond=K)
    x_star = exact.dense_solve(G, b)
    assert pc.converged and pc.iterations < hs.iterations
    assert rel(pc.x, x_star) <= 1e-8
    assert abs(sp1.iterations - pc.iterations) <= 1 and rel(sp1.x, x_star) <= 1e-8


def test_block_jacobi_blocks_are_the_pixel_blocks_of_G():
    """The oracle extracts K_j from the assembled G; the pixel block of G = B^T C B + Q at pixel j is
    h_j A^T T A + diag(Q0)_jj P (Eq.(7), Q = P (x) Q0), with diag(Q0)_jj = kappa2 + deg_j for the
    Laplacian prior (deg 2 at corners, 3 on edges, 4 inside: P:L100-106).  Checked on a patch with
    random hits by applying the preconditioner to unit vectors."""
    p = make_patch(3, 6, 3, seed=4, hits="random")
    K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits)
    side, N, k = p.side, p.N, p.k
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    h = np.asarray(p.hits).reshape(N)
    for j in (0, side - 1, 1, side + 1, N - 1, 3 * side + 4):
        y, x = divmod(j, side)
        deg = 4 - (y == 0) - (y == side - 1) - (x == 0) - (x == side - 1)
        Kj = h[j] * M + (p.kappa2 + deg) * np.diag(p.tau)
        for c in range(k):
            e = np.zeros(k * N)
            e[c * N + j] = 1.0
            z = K(e).reshape(k, N)
            assert np.allclose(z[:, j], np.linalg.solve(Kj, np.eye(k)[c]), rtol=1e-12, atol=0)
            z[:, j] = 0.0
            assert not z.any()                      # block diagonal: nothing leaks to other pixels


def test_exact_preconditioner_converges_in_one_iteration(tiny):
    """PCG with K = G (z = G^{-1} r by a direct solve) converges in one step (Saad Alg. 9.1)."""
    p, G, b = tiny
    import scipy.sparse.linalg as sl
    lu = sl.splu(G.tocsc())
    for fn in (cg.cg_hs, cg.cg_single_pass):
        res = fn(G, b, tol=1e-10, precond=lu.solve)
        assert res.converged and res.iterations == 1


def test_breakdown_detected_on_indefinite():
    import scipy.sparse as sp
    G = sp.diags([1.0, -1.0, 2.0]).tocsr()
    b = np.array([1.0, 1.0, 0.0])
    assert cg.cg_hs(G, b).status == "breakdown"


@pytest.mark.slow
def test_cg_medium_matches_dct_exact():
    p = make_config("medium")[0]
    G, b = model.problem_system(p)
    res = cg.cg_hs(G, b, tol=1e-10)
    x_star = exact.problem_dct_exact(p)
    assert res.converged
    assert rel(res.x, x_star) <= 1e-8


@pytest.mark.parametrize("prior", ["d2"])
def test_cg_d2_prior_small(prior):
    p = make_patch(4, 9, 3, seed=9, prior=prior)
    G, b = model.problem_system(p)
    res = cg.cg_hs(G, b, tol=1e-10)
    assert res.converged
    assert rel(res.x, exact.problem_dct_exact(p)) <= 1e-8
    assert rel(res.x, exact.dense_solve(G, b)) <= 1e-8


def test_warm_start_pins(tiny):
    """Warm start (reading R37), pinned to the plain definitions: x0 = 0 is the cold start bit for
    bit; x0 = the dense solution stops before the first step; any x0 reaches the dense solution
    within the tolerance's reach; CG from x0 on (b) equals CG from 0 on b - G x0 shifted by x0 (the
    textbook identity behind r_0 = b - G x_0)."""
    _, G, b = tiny
    x_star = exact.dense_solve(G, b)
    cold = cg.cg_hs(G, b, tol=1e-10)
    zero = cg.cg_hs(G, b, tol=1e-10, x0=np.zeros_like(b))
    assert zero.iterations == cold.iterations and np.array_equal(zero.x, cold.x)
    at = cg.cg_hs(G, b, tol=1e-10, x0=x_star)
    assert at.iterations == 0 and at.converged and np.array_equal(at.x, x_star)
    rng = np.random.default_rng(3)
    x0 = x_star + 1e-3 * np.linalg.norm(x_star) / np.sqrt(b.size) * rng.standard_normal(b.size)
    w = cg.cg_hs(G, b, tol=1e-10, x0=x0)
    assert w.converged and np.linalg.norm(G @ w.x - b) <= 1.5e-10 * np.linalg.norm(b)
    assert np.linalg.norm(w.x - x_star) <= 1e-6 * np.linalg.norm(x_star)
    assert w.iterations < cold.iterations               # a good guess saves steps
    # shifted system: same iterates up to rounding, same counts (the rule is relative to ||b||)
    d = b - G @ x0
    sh = cg.cg_hs(G, d, tol=1e-10 * np.linalg.norm(b) / np.linalg.norm(d))
    assert abs(sh.iterations - w.iterations) <= 1
    assert np.linalg.norm((x0 + sh.x) - w.x) <= 1e-9 * np.linalg.norm(x_star)
    # b = 0: the rule falls back to ||r_0|| and CG drives x0 to the solution 0
    z = cg.cg_hs(G, np.zeros_like(b), tol=1e-8, x0=x0)
    assert z.converged and np.linalg.norm(z.x) <= 1e-6 * np.linalg.norm(x0)
