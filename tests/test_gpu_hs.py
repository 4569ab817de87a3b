"""GPU parity of the textbook Hestenes-Stiefel CG variant (desc.cg_variant = KCG_CG_HS; reading R9, the
paper's "two variants of the conjugate gradient approach") against the oracle's textbook
HS-CG (oracle/cg.py cg_hs, Alg. CG P:L225-241 read per R7/R8) -- like for like: same algorithm, so
the iterates agree to rounding and the iteration counts within +-2 (bar of BASELINE north_star)."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, oracle_count_envelope, rel
from oracle import cg, exact, model, sylvester
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
TOL = 1e-10


def _check(ps, precond=None, **kw):
    ctx, Y = make_ctx(ps, cg_variant="hs", precond=precond or "none", **kw)
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    mu = mu.cpu().numpy()
    assert rep["converged"], rep["status_name"]
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        K = None
        if precond:
            K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits, p.prior)
        lo, hi, ref = oracle_count_envelope(cg.cg_hs, G, b, tol=TOL, precond=K, max_iter=200000)
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        assert lo - 2 <= rep["iterations_per"][i] <= hi + 2, (i, rep["iterations_per"][i], lo, hi)
    assert rep["rel_residual_true"] <= 5 * TOL
    return ctx, Y, mu, rep


def test_hs_tiny_medium():
    _check(make_config("tiny"))
    _check(make_config("medium"))


@pytest.mark.parametrize("level,k,hits", [(0, 1, None), (0, 3, None), (1, 2, "random"), (2, 3, None),
                                          (3, 4, "random"), (4, 5, None), (5, 6, "random"), (6, 8, None),
                                          (7, 2, None), (6, 7, "random")])
def test_hs_edge_levels(level, k, hits):
    _check([make_patch(level, 9, k, seed=600 + s, tau="loguniform", hits=hits) for s in range(2)])


@pytest.mark.parametrize("level,k,hits", [(3, 3, None), (5, 4, "random"), (6, 1, None)])
def test_hs_d2(level, k, hits):
    _check([make_patch(level, 9, k, seed=620 + s, tau="loguniform", prior="d2", hits=hits) for s in range(2)])


@pytest.mark.parametrize("level,k,hits,prior", [(0, 2, None, "laplacian"), (4, 4, "random", "laplacian"),
                                                (5, 7, None, "laplacian"), (5, 3, "random", "d2")])
def test_hs_block_jacobi(level, k, hits, prior):
    _check([make_patch(level, 9, k, seed=640 + s, tau="loguniform", hits=hits, prior=prior) for s in range(2)],
           precond="block_jacobi")


def test_hs_planck_vs_exact_and_variants_agree():
    p = make_config("planck")[0]
    ctx, Y = make_ctx([p], cg_variant="hs")
    mu, rep = ctx.solve(Y, tol=TOL)
    assert rep["converged"] and rep["rel_residual_true"] <= 2 * TOL
    assert rel(mu.cpu().numpy()[0], exact.problem_dct_exact(p)) <= 1e-8
    c1, _ = make_ctx([p])
    mu1, rep1 = c1.solve(Y, tol=TOL)
    assert abs(rep1["iterations"] - rep["iterations"]) <= 2
    assert rel(mu1.cpu().numpy(), mu.cpu().numpy()) <= 1e-8
    # loop bytes: 72 K N per iteration (56 for the first, x not yet updated)
    k, N, it = p.k, p.N, rep["iterations"]
    assert rep["loop_bytes"] == (56.0 * it + 16.0 * (it - 1)) * k * N


def test_hs_sylvester_and_kohler():
    ps = [make_patch(6, 9, 4, seed=660 + s, tau="loguniform", hits=h) for s, h in enumerate([None, "random"])]
    ctx, Y = make_ctx(ps, cg_variant="hs")
    mu, rep = ctx.sylvester(Y, tol=TOL)
    mu = mu.cpu().numpy()
    for i, p in enumerate(ps):
        ref = sylvester.problem_solve(p, tol=TOL)
        assert rel(mu[i], ref.x) <= 1e-8
        gits = rep["iterations_per"][i * 4:(i + 1) * 4]
        assert all(abs(a - b) <= 2 for a, b in zip(gits, ref.iterations)), (gits, ref.iterations)
    from oracle import kohler
    mk, repk = ctx.kohler(Y, tol=TOL)
    mk = mk.cpu().numpy()
    for i, p in enumerate(ps):
        ref = kohler.problem_solve(p, tol=TOL)
        assert rel(mk[i], ref.x) <= 1e-8


def test_hs_zero_rhs_max_iter_and_nonfinite():
    import torch
    from paper_2204_08057_b200.kroncg import KcgError
    ps = [make_patch(5, 9, 3, seed=1)]
    ctx, Y = make_ctx(ps, cg_variant="hs")
    mu, rep = ctx.solve(torch.zeros_like(Y), tol=TOL)
    assert rep["iterations"] == 0 and rep["converged"] and not mu.any()
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=7)
    assert rep["status_name"] == "KCG_NOT_CONVERGED" and rep["iterations"] == 7
    G, b = model.problem_system(ps[0])
    ref = cg.cg_hs(G, b, tol=1e-30, max_iter=7)
    assert rel(mu.cpu().numpy()[0], ref.x) <= 1e-10
    Y[0, 1, 2, 2] = float("nan")
    with pytest.raises(KcgError) as e:
        ctx.solve(Y, tol=TOL)
    assert e.value.status == 5


def test_hs_fullsky_batch_vs_oracle_counts():
    """12 faces in one launch, per-face freeze; counts against the committed oracle HS counts."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "oracle_iterations.json")) as f:
        golden = json.load(f)["fullsky"]["kron_cg_iterations"]
    ps = make_config("fullsky")
    ctx, Y = make_ctx(ps, cg_variant="hs")
    mu, rep = ctx.solve(Y, tol=TOL)
    mu = mu.cpu().numpy()
    assert rep["converged"]
    for i, p in enumerate(ps):
        assert abs(rep["iterations_per"][i] - golden[i]) <= 2, (i, rep["iterations_per"][i], golden[i])
        assert rel(mu[i], exact.problem_dct_exact(p)) <= 1e-8
