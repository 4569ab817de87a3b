"""Pins for oracle.variance (posterior variances, reading R32)."""

import numpy as np
import pytest

from oracle import exact, model, variance
from synth import make_patch


def test_splitmix64_reference_output():
    # first output of Vigna's reference SplitMix64 seeded with 0 (state 0 -> 0xE220A8397B1DCDAF)
    assert int(variance.splitmix64(0)) == 0xE220A8397B1DCDAF
    # and it is a function of the state only (vectorised == scalar)
    xs = np.arange(5, dtype=np.uint64)
    assert [int(v) for v in variance.splitmix64(xs)] == [int(variance.splitmix64(int(x))) for x in xs]


def test_rademacher_probes_are_balanced_and_seeded():
    z = variance.rademacher(7, 0, 3, 4, 4096)
    assert z.shape == (3, 4, 4096) and set(np.unique(z)) == {-1.0, 1.0}
    assert abs(z.mean()) < 4 / np.sqrt(z.size)
    assert np.array_equal(z, variance.rademacher(7, 0, 3, 4, 4096))
    assert not np.array_equal(z, variance.rademacher(7, 1, 3, 4, 4096))
    assert not np.array_equal(z, variance.rademacher(8, 0, 3, 4, 4096))
    # distinct probes are uncorrelated: E[z_i z_j] = delta_ij
    c = (variance.rademacher(7, 0, 1, 1, 20000) * variance.rademacher(7, 1, 1, 1, 20000)).mean()
    assert abs(c) < 4 / np.sqrt(20000)


def test_exact_diag_matches_dct_mode_sum():
    """hits = 1, k = 1: diag((M + phi (kappa2 + L))^{-1}) = sum_ab v_ab(j)^2 / (m + phi (kappa2 + lam_ab))."""
    p = make_patch(3, 2, 1, seed=4, tau="given", tau_values=[3.0])
    G, _ = model.problem_system(p)
    d = variance.exact_diag(G)
    s = p.side
    t = 2.0 - 2.0 * np.cos(np.pi * np.arange(s) / s)
    m = float(p.A[:, 0] @ (p.noise_prec * p.A[:, 0]))
    u = np.sqrt(2.0 / s) * np.cos(np.pi * np.outer(np.arange(s) + 0.5, np.arange(s)) / s)
    u[:, 0] = np.sqrt(1.0 / s)                           # orthonormal DCT-II basis, u[y, a]
    den = m + 3.0 * (p.kappa2 + t[:, None] + t[None, :])  # [a, b]
    ref = np.einsum("ya,xb,ab->yx", u ** 2, u ** 2, 1.0 / den).reshape(-1)
    assert np.allclose(d, ref, rtol=1e-12)


@pytest.mark.parametrize("hits", [None, "random"])
def test_hutchinson_is_unbiased_within_its_standard_error(hits):
    """With exact solves, |est - diag(G^-1)| <= 5 sigma entrywise, sigma^2 = (1/s) sum_{l != j} Ginv_jl^2."""
    p = make_patch(3, 9, 3, seed=12, tau="loguniform", hits=hits)
    G, _ = model.problem_system(p)
    Gi = np.linalg.inv(G.toarray())
    s = 400
    est = variance.hutchinson([G], p.k, p.N, s, seed=3, solve=lambda A, z: Gi @ z)[0]
    d = np.diag(Gi)
    sig = np.sqrt((np.sum(Gi ** 2, axis=1) - d ** 2) / s)
    z = np.abs(est - d) / sig
    assert z.max() <= 5.0, z.max()
    assert 0.5 < np.sqrt(np.mean(z ** 2)) < 1.5           # the error scale is the predicted one


def test_hutchinson_with_cg_equals_exact_solves():
    p = make_patch(3, 9, 3, seed=13, tau="loguniform")
    G, _ = model.problem_system(p)
    a = variance.hutchinson([G], p.k, p.N, 4, seed=9)
    b = variance.hutchinson([G], p.k, p.N, 4, seed=9, solve=lambda A, z: exact.dense_solve(A, z))
    assert np.abs(a - b).max() <= 1e-8 * np.abs(b).max()


def test_dct_diag_moments_match_the_dense_inverse():
    p = make_patch(3, 9, 3, seed=14, tau="loguniform")
    G, _ = model.problem_system(p)
    Gi = np.linalg.inv(G.toarray())
    d1, d2 = variance.dct_diag_moments(p.level, p.A, p.noise_prec, p.tau, p.kappa2)
    assert np.allclose(d1.reshape(-1), np.diag(Gi), rtol=1e-11)
    assert np.allclose(d2.reshape(-1), np.sum(Gi ** 2, axis=1), rtol=1e-11)
