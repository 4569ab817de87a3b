"""GPU parity of Alg. Kohler (sylvester_kohler_solve) against the
oracle's step-by-step implementation (oracle/kohler.py, same canonical Schur factor) and the exact
solutions.  Bar: relative error <= 1e-8 against the oracle at tol 1e-10, per-column iterations +-2."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from oracle import exact, kohler, model
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
TOL = 1e-10


def _check(ps, **kw):
    ctx, Y = make_ctx(ps, **kw)
    mu, rep = ctx.kohler(Y, tol=TOL)
    mu = mu.cpu().numpy()
    assert rep["converged"], rep
    k = ps[0].k
    for i, p in enumerate(ps):
        ref = kohler.problem_solve(p, tol=TOL)
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        for c in range(k):
            assert abs(rep["iterations_per"][i * k + c] - ref.iterations[c]) <= 2
    return mu, rep


def test_kohler_tiny_medium_vs_oracle_and_exact():
    for name in ("tiny", "medium"):
        ps = make_config(name)
        mu, rep = _check(ps)
        assert rel(mu[0], exact.problem_dct_exact(ps[0])) <= 1e-8


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 8])
def test_kohler_every_k_batched(k):
    _check([make_patch(5, 9, k, seed=800 + 9 * k + s, tau="loguniform") for s in range(3)])


@pytest.mark.parametrize("prior,hits", [("laplacian", "random"), ("d2", None), ("d2", "random")])
def test_kohler_hits_and_d2(prior, hits):
    _check([make_patch(6, 9, 4, seed=820 + s, tau="loguniform", prior=prior, hits=hits) for s in range(2)])


def test_kohler_planck_vs_exact_and_routes_agree():
    ps = make_config("planck")
    ctx, Y = make_ctx(ps)
    mu, rep = ctx.kohler(Y, tol=TOL)
    assert rep["converged"]
    ex = exact.problem_dct_exact(ps[0])
    assert rel(mu.cpu().numpy()[0], ex) <= 1e-8
    mu2, _ = ctx.sylvester(Y, tol=TOL)
    assert rel(mu.cpu().numpy(), mu2.cpu().numpy()) <= 1e-8


def test_kohler_nested_is_a_permutation():
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.problems import stack
    p = make_patch(6, 9, 3, seed=840, tau="loguniform", hits="random")
    ctx_r, Y = make_ctx([p])
    mu_r, _ = ctx_r.kohler(Y, tol=TOL)
    st = stack([p])
    nest = lambda a: model.to_layout(p.level, a, "nested").reshape(np.shape(a))
    ctx_n = KronCG(p.level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                   hits=torch.from_numpy(nest(st["hits"])).cuda(), layout="nested")
    mu_n, _ = ctx_n.kohler(torch.from_numpy(nest(st["Y"])).cuda(), tol=TOL)
    assert np.array_equal(mu_n.cpu().numpy(), nest(mu_r.cpu().numpy()))


def test_kohler_with_block_jacobi_columns():
    """precond = block_jacobi: each column's shifted system preconditioned by its diagonal (the
    k = 1 block Jacobi); same solution as the oracle's unpreconditioned Kohler to the tolerance."""
    ps = [make_patch(6, 9, 4, seed=850 + s, tau="loguniform", hits="random") for s in range(2)]
    ctx, Y = make_ctx(ps, precond="block_jacobi")
    mu, rep = ctx.kohler(Y, tol=TOL)
    assert rep["converged"]
    for i, p in enumerate(ps):
        assert rel(mu.cpu().numpy()[i], kohler.problem_solve(p, tol=TOL).x) <= 1e-8
