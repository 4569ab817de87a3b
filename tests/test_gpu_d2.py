"""GPU parity of the paper's D^2 prior (Q0 = D^2 + kappa2 I, reading R3 "d2"; SURVEY 8(f)
NEXT-2): radius-2 operator, single-pass CG with a 4-pixel halo, against the oracle's literal
assembly (D @ D) and the DCT-exact solve (D^2 -> lambda^2)."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, oracle_count_envelope, rel
from oracle import cg, exact, model, sylvester
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

TOL = 1e-10


def _d2(level, k, seed, **kw):
    return make_patch(level, 9, k, seed=seed, tau="loguniform", prior="d2", **kw)


@pytest.mark.parametrize("level,k,hits", [(0, 1, None), (1, 2, None), (2, 3, "random"), (3, 4, None),
                                          (5, 4, "random"), (6, 1, None), (7, 3, None)])
def test_d2_kron_vs_oracle(level, k, hits):
    ps = [_d2(level, k, 170 + s, hits=hits) for s in range(2)]
    ctx, Y = make_ctx(ps)
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    mu = mu.cpu().numpy()
    assert rep["converged"], rep
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        ref = cg.cg_hs(G, b, tol=TOL, max_iter=200000)
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        # iteration counts like-for-like (reading R9): the D^2 faces of level <= 3 need more CG steps
        # than unknowns, a rounding-dominated regime where even the oracle's HS and single-pass
        # variants differ by up to 9 steps
        # -> the GPU count must lie in the envelope of the two oracle variants +- 2 (which is +- 2
        # around both when they agree, as they do once CG needs far fewer steps than unknowns)
        sp = cg.cg_single_pass(G, b, tol=TOL, max_iter=200000)
        lo, hi = min(ref.iterations, sp.iterations) - 2, max(ref.iterations, sp.iterations) + 2
        assert lo <= rep["iterations_per"][i] <= hi, (rep["iterations_per"][i], ref.iterations, sp.iterations)
    assert rep["rel_residual_true"] <= 5 * TOL


@pytest.mark.parametrize("level,k,hits", [(0, 1, None), (1, 2, None), (2, 3, "random"), (3, 4, None),
                                          (5, 4, "random"), (6, 1, None), (7, 3, None)])
def test_d2_variants_like_for_like(level, k, hits):
    """Reading R9 like for like: the GPU's textbook HS variant against the oracle's HS-CG and the GPU's
    single-pass kernel against the oracle's single-pass CG, each at 1e-8 and +-2 iterations around the
    oracle's rounding envelope (reading R34: at levels <= 3 CG needs almost as many steps as there
    are unknowns and the oracle's own count moves by up to 2 under a 2^-50 change of b)."""
    ps = [_d2(level, k, 170 + s, hits=hits) for s in range(2)]
    for variant, fn in (("hs", cg.cg_hs), ("single_pass", cg.cg_single_pass)):
        ctx, Y = make_ctx(ps, cg_variant=variant)
        mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
        mu = mu.cpu().numpy()
        assert rep["converged"], rep
        for i, p in enumerate(ps):
            G, b = model.problem_system(p)
            lo, hi, ref = oracle_count_envelope(fn, G, b, tol=TOL, max_iter=200000)
            assert rel(mu[i], ref.x) <= 1e-8, (variant, i, rel(mu[i], ref.x))
            assert lo - 2 <= rep["iterations_per"][i] <= hi + 2, (variant, rep["iterations_per"][i], lo, hi)


def test_d2_apply_matches_assembled():
    import torch
    ps = [_d2(6, 4, 180, hits="random"), _d2(6, 4, 181)]
    ctx, _ = make_ctx(ps)
    x = np.random.default_rng(1).standard_normal((2, 4, 64, 64))
    y = ctx.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    for i, p in enumerate(ps):
        G, _ = model.problem_system(p)
        ref = G @ x[i].reshape(-1)
        assert np.allclose(y[i].reshape(-1), ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


def test_d2_medium_vs_exact_sylvester_and_pcg():
    p = make_config("medium", prior="d2")[0]
    ctx, Y = make_ctx([p])
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    xe = exact.problem_dct_exact(p)
    assert rep["converged"] and rel(mu.cpu().numpy()[0], xe) <= 1e-8
    mu2, rep2 = ctx.sylvester(Y, tol=TOL, max_iter=200000)
    sref = sylvester.problem_solve(p, tol=TOL, max_iter=200000)
    assert rel(mu2.cpu().numpy()[0], sref.x) <= 1e-8
    c3, Y3 = make_ctx([p], precond="block_jacobi")
    mu3, rep3 = c3.solve(Y3, tol=TOL, max_iter=200000)
    K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2, prior="d2")
    ref3 = cg.cg_hs(*model.problem_system(p), tol=TOL, max_iter=200000, precond=K)
    assert rel(mu3.cpu().numpy()[0], ref3.x) <= 1e-8 and abs(rep3["iterations"] - ref3.iterations) <= 2
    assert rep3["iterations"] < rep["iterations"]


def test_d2_planck_vs_exact():
    p = make_config("planck", prior="d2")[0]
    ctx, Y = make_ctx([p])
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    assert rep["converged"] and rel(mu.cpu().numpy()[0], exact.problem_dct_exact(p)) <= 1e-8


def test_d2_limits():
    from paper_2204_08057_b200.kroncg import KcgError
    with pytest.raises(KcgError) as e:
        make_ctx([_d2(4, 5, 1)])
    assert e.value.status == 4


@pytest.mark.parametrize("level,k", [(5, 4), (6, 2), (7, 3)])
def test_d2_block_jacobi_with_hits(level, k):
    """The row-march kernel's block-Jacobi path with per-pixel Cholesky (hits): u = K^{-1} r over every
    plane of the stage (A) and over the shared r_new rows (B'), C0 / C1 one row further behind --
    Kronecker route (K = 4: two planes per warp, K = 2 / 3: one) and the Sylvester columns (K = 1:
    two face columns per lane) against the oracle's preconditioned CG (reading R10)."""
    ps = [_d2(level, k, 860 + s, hits="random") for s in range(2)]
    ctx, Y = make_ctx(ps, precond="block_jacobi")
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    mu = mu.cpu().numpy()
    assert rep["converged"], rep["status_name"]
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits, prior="d2")
        lo, hi, ref = oracle_count_envelope(cg.cg_hs, G, b, tol=TOL, precond=K, max_iter=200000)
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        sp = cg.cg_single_pass(G, b, tol=TOL, max_iter=200000, precond=K)
        assert min(lo, sp.iterations) - 2 <= rep["iterations_per"][i] <= max(hi, sp.iterations) + 2
    smu, srep = ctx.sylvester(Y, tol=TOL, max_iter=200000)
    smu = smu.cpu().numpy()
    assert srep["converged"]
    for i, p in enumerate(ps):
        ref = sylvester.problem_solve(p, tol=TOL, max_iter=200000, precond="jacobi")
        assert rel(smu[i], ref.x) <= 1e-8, (i, rel(smu[i], ref.x))


def test_d2_march_ragged_strips_and_segments():
    """Face widths that are not multiples of the strips (56 output columns for K = 4 and K = 1) and a
    Sylvester route with several segments per strip: level 8 (256 = 10 x 24 + 16 = 4 x 56 + 32)."""
    p = _d2(8, 4, 880)
    ctx, Y = make_ctx([p])
    mu, rep = ctx.solve(Y, tol=TOL, max_iter=200000)
    xe = exact.problem_dct_exact(p)
    assert rep["converged"] and rel(mu.cpu().numpy()[0], xe) <= 1e-8
    smu, srep = ctx.sylvester(Y, tol=TOL, max_iter=200000)
    assert srep["converged"] and rel(smu.cpu().numpy()[0], xe) <= 1e-8
    kmu, krep = ctx.kohler(Y, tol=TOL, max_iter=200000)
    assert krep["converged"] and rel(kmu.cpu().numpy()[0], xe) <= 1e-8


@pytest.mark.parametrize("k,hits", [(4, None), (4, "random"), (1, None)])
def test_d2_march_batch_independent_bitwise(k, hits):
    """The row march re-plans its segment length every pass from the number of systems still running
    (kcg::m_seg_model), and its partials are per (strip, 16-row block), so a face's iterate must not
    depend on the batch it is solved in: face 0 alone (one system: short segments) and inside a batch
    of four faces of different conditioning (longer segments, faces leaving at different passes) agree
    bit for bit, and both equal the oracle at 1e-8."""
    ps = [_d2(8, k, 510 + s, hits=hits) for s in range(4)]
    ctx1, Y1 = make_ctx(ps[:1])
    mu1, rep1 = ctx1.solve(Y1, tol=TOL, max_iter=200000)
    ctx4, Y4 = make_ctx(ps)
    mu4, rep4 = ctx4.solve(Y4, tol=TOL, max_iter=200000)
    assert rep1["converged"] and rep4["converged"]
    assert len(set(rep4["iterations_per"])) > 1, rep4["iterations_per"]  # faces leave at different passes
    a, b = mu1.cpu().numpy()[0], mu4.cpu().numpy()[0]
    assert rep1["iterations_per"][0] == rep4["iterations_per"][0]
    assert np.array_equal(a, b), float(np.abs(a - b).max())
    G, bb = model.problem_system(ps[0])
    ref = cg.cg_hs(G, bb, tol=TOL, max_iter=200000)
    assert rel(a, ref.x) <= 1e-8
