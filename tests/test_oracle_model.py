"""Pins for oracle.model: the assembled G and b against the posterior written entrywise,
closed-form special cases and the DCT eigenmodes."""

import numpy as np
import pytest
from scipy.fft import idctn

from oracle import grid, model
from synth import make_patch


def test_scalar_case():
    # SPEC S:L212 / S:L430: n = m = 1, single pixel (L = 0, D = 0): G = tau a^2 h + phi kappa2.
    A = np.array([[1.7]])
    T = np.array([3.0])
    tau = np.array([5.0])
    G = model.assemble_G(0, A, T, tau, 0.25, hits=np.array([2.0]))
    assert G.shape == (1, 1)
    assert np.isclose(G[0, 0], 3.0 * 1.7 ** 2 * 2.0 + 5.0 * 0.25, rtol=1e-15)
    b = model.assemble_rhs(0, A, T, np.array([[[0.5]]]), hits=np.array([2.0]))
    assert np.isclose(b[0], 1.7 * 3.0 * 2.0 * 0.5, rtol=1e-15)


@pytest.mark.parametrize("prior", ["laplacian", "d2"])
@pytest.mark.parametrize("hits", [None, "random"])
def test_G_b_are_hessian_and_gradient_of_posterior(prior, hits):
    # Eq.(Q*)/(mu*): -log p(S|Y) = 1/2 S^T G S - b^T S + c.  Polarisation recovers G and b
    # exactly from the entrywise likelihood Eq.(2) + prior Eq.(3).
    p = make_patch(1, 3, 2, seed=7, tau="given", tau_values=[2.0, 30.0], prior=prior,
                   hits=hits)
    G = model.assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits, prior).toarray()
    b = model.assemble_rhs(p.level, p.A, p.noise_prec, p.Y, p.hits)
    dim = p.k * p.N

    def f(vecS):
        return model.neg_log_posterior(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.Y,
                                       vecS.reshape(p.k, p.N), p.hits, prior)

    E = np.eye(dim)
    f0 = f(np.zeros(dim))
    fe = [f(E[i]) for i in range(dim)]
    Gref = np.empty((dim, dim))
    for i in range(dim):
        Gref[i, i] = f(2 * E[i]) - 2 * fe[i] + f0
        for j in range(i + 1, dim):
            Gref[i, j] = Gref[j, i] = f(E[i] + E[j]) - fe[i] - fe[j] + f0
    bref = np.array([(f(-E[i]) - fe[i]) / 2 for i in range(dim)])
    scale = np.abs(G).max()
    assert np.abs(G - Gref).max() <= 1e-9 * scale
    assert np.abs(b - bref).max() <= 1e-9 * np.abs(b).max()


@pytest.mark.parametrize("prior", ["laplacian", "d2"])
def test_dct_eigenmodes(prior):
    # G (v_ab (x) c) = v_ab (x) (M + lam^{Q0}_ab P) c, v_ab a 2-D DCT-II basis vector.
    level = 3
    p = make_patch(level, 5, 3, seed=3, tau="given", tau_values=[1.0, 7.0, 40.0],
                   prior=prior)
    s = p.side
    G = model.assemble_G(level, p.A, p.noise_prec, p.tau, p.kappa2, None, prior)
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    P = np.diag(p.tau)
    t = 2 - 2 * np.cos(np.pi * np.arange(s) / s)
    rng = np.random.default_rng(0)
    for (a, bb) in [(0, 0), (1, 0), (0, 5), (3, 7), (7, 7)]:
        e = np.zeros((s, s))
        e[a, bb] = 1.0
        v = idctn(e, type=2, norm="ortho").ravel()
        lam = t[a] + t[bb]
        lq = p.kappa2 + (lam if prior == "laplacian" else lam * lam)
        c = rng.standard_normal(3)
        x = np.kron(c, v)
        y = G @ x
        ref = np.kron((M + lq * P) @ c, v)
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("prior", ["laplacian", "d2"])
def test_rows_one_by_one_match_assembly(prior):
    p = make_patch(4, 9, 4, seed=11, tau="loguniform", prior=prior, hits="random")
    G = model.assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits, prior)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((p.k, p.N))
    full = G @ x.ravel()
    rows = [(int(rng.integers(p.k)), int(rng.integers(p.N))) for _ in range(40)]
    rows += [(0, 0), (3, p.N - 1), (1, p.side - 1), (2, p.N - p.side)]
    got = model.apply_G_rows(p.level, p.A, p.noise_prec, p.tau, p.kappa2, x, rows, p.hits, prior)
    ref = np.array([full[l * p.N + j] for (l, j) in rows])
    assert np.allclose(got, ref, rtol=1e-13, atol=1e-13 * np.abs(full).max())


def test_spd_and_symmetric():
    p = make_patch(3, 9, 3, seed=0)
    G = model.assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2).toarray()
    assert np.array_equal(G, G.T)
    assert np.linalg.eigvalsh(G).min() > 0
    # Q alone is only PSD with kappa2 = 0: one zero eigenvalue per source
    Q = model.Q_matrix(p.level, p.tau, 0.0).toarray()
    ev = np.linalg.eigvalsh(Q)
    assert np.sum(np.abs(ev) < 1e-10 * ev.max()) == p.k


def test_constant_data_gives_constant_mean():
    # Y_j = y for all j: mu is constant = (M + kappa2 P)^{-1} A^T T y (L 1 = 0).
    p = make_patch(3, 6, 3, seed=5)
    y = np.array([0.3, -1.0, 2.0, 0.5, 0.1, 1.5])
    Y = np.repeat(y[:, None], p.N, axis=1).reshape(6, p.side, p.side)
    G = model.assemble_G(p.level, p.A, p.noise_prec, p.tau, p.kappa2)
    b = model.assemble_rhs(p.level, p.A, p.noise_prec, Y)
    mu = np.linalg.solve(G.toarray(), b).reshape(3, p.N)
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    ref = np.linalg.solve(M + p.kappa2 * np.diag(p.tau), p.A.T @ (p.noise_prec * y))
    assert np.allclose(mu, ref[:, None], rtol=1e-10, atol=1e-12)


def test_nested_system_solution_is_the_permuted_row_major_one():
    """The posterior mean does not depend on the pixel numbering: solving the NESTED-ordered system
    gives the row-major solution permuted pixel-wise (each source plane)."""
    from oracle import exact, grid
    p = make_patch(3, 9, 3, seed=5, tau="loguniform", hits="random")
    Gr, br = model.problem_system(p)
    Gn, bn = model.problem_system(p, layout="nested")
    xr = exact.dense_solve(Gr, br).reshape(p.k, -1)
    xn = exact.dense_solve(Gn, bn).reshape(p.k, -1)
    perm = grid.pixel_index(p.level, "nested").reshape(-1)
    assert np.allclose(xn[:, perm], xr, rtol=1e-12, atol=1e-12 * np.abs(xr).max())
