"""GPU parity of the many-right-hand-side entry points: kron_cg_solve_b for
given b, parameter sweeps as batched patches, and the Hutchinson posterior variances
(posterior_variance) against the oracle with the SAME counter-based probes (oracle/variance.py)."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from oracle import cg, model, variance
from synth import make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
TOL = 1e-10


@pytest.mark.parametrize("layout,hits", [("row", None), ("row", "random"), ("nested", "random")])
def test_solve_b_vs_oracle(layout, hits):
    import torch
    ps = [make_patch(5, 9, 3, seed=500 + s, tau="loguniform", hits=hits) for s in range(3)]
    kw = {}
    if layout == "nested":
        from synth.problems import stack
        from paper_2204_08057_b200.kroncg import KronCG
        st = stack(ps)
        nest = lambda a: model.to_layout(5, a, "nested").reshape(np.shape(a))
        ctx = KronCG(5, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                     hits=torch.from_numpy(nest(st["hits"])).cuda(), layout="nested")
    else:
        ctx, _ = make_ctx(ps)
    rng = np.random.default_rng(1)
    b = rng.standard_normal((3, 3, 32, 32))
    x, rep = ctx.solve_b(torch.from_numpy(b).cuda(), tol=TOL)
    x = x.cpu().numpy()
    assert rep["converged"] and rep["rel_residual_true"] <= 2e-10
    for i, p in enumerate(ps):
        G, _ = model.problem_system(p, layout=layout)
        ref = cg.cg_hs(G, b[i].reshape(-1), tol=TOL)
        assert rel(x[i].reshape(-1), ref.x) <= 1e-8
        assert abs(rep["iterations_per"][i] - ref.iterations) <= 2


def test_parameter_sweep_is_one_batched_launch():
    """INLA-style sweep: one data set, a grid of (kappa2, tau) -- 16 parameter sets as 16
    patches of one context, solved in one launch, each against its own oracle solve."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    base = make_patch(5, 9, 3, seed=520, tau="loguniform")
    grid = [(k2, sc) for k2 in (0.01, 0.1, 1.0, 10.0) for sc in (0.1, 1.0, 10.0, 100.0)]
    P = len(grid)
    A = np.stack([base.A] * P)
    T = np.stack([base.noise_prec] * P)
    tau = np.stack([base.tau * sc for _, sc in grid])
    k2 = np.array([k for k, _ in grid])
    ctx = KronCG(5, A, T, tau, k2)
    Y = torch.from_numpy(np.stack([base.Y] * P)).cuda()
    mu, rep = ctx.solve(Y, tol=TOL)
    mu = mu.cpu().numpy()
    assert rep["converged"]
    for i, (kk, sc) in enumerate(grid):
        G = model.assemble_G(5, base.A, base.noise_prec, base.tau * sc, kk)
        b = model.assemble_rhs(5, base.A, base.noise_prec, base.Y)
        ref = cg.cg_hs(G, b, tol=TOL)
        assert rel(mu[i].reshape(-1), ref.x) <= 1e-8


@pytest.mark.parametrize("layout,hits", [("row", None), ("row", "random"), ("nested", None)])
def test_posterior_variance_matches_oracle_hutchinson(layout, hits):
    """Same probes on both sides: the GPU estimate equals the oracle's to CG accuracy."""
    import torch
    ps = [make_patch(5, 9, 3, seed=540 + s, tau="loguniform", hits=hits) for s in range(2)]
    if layout == "nested":
        from synth.problems import stack
        from paper_2204_08057_b200.kroncg import KronCG
        st = stack(ps)
        ctx = KronCG(5, st["A"], st["noise_prec"], st["tau"], st["kappa2"], layout="nested")
    else:
        ctx, _ = make_ctx(ps)
    s = 6
    var, rep = ctx.posterior_variance(s, seed=77, tol=TOL)
    var = var.cpu().numpy().reshape(2, -1)
    systems = [model.problem_system(p, layout=layout)[0] for p in ps]
    ref = variance.hutchinson(systems, 3, ps[0].N, s, seed=77, tol=TOL)
    assert np.abs(var - ref).max() <= 1e-8 * np.abs(ref).max()


def test_posterior_variance_converges_to_the_exact_diagonal():
    """Many probes on a small face: within 5 sigma of diag(G^-1) (dense inverse) everywhere."""
    p = make_patch(3, 9, 2, seed=560, tau="loguniform")
    ctx, _ = make_ctx([p])
    s = 256
    var, rep = ctx.posterior_variance(s, seed=5, tol=1e-12)
    var = var.cpu().numpy().reshape(-1)
    G, _ = model.problem_system(p)
    Gi = np.linalg.inv(G.toarray())
    d = np.diag(Gi)
    sig = np.sqrt((np.sum(Gi ** 2, axis=1) - d ** 2) / s)
    assert (np.abs(var - d) / sig).max() <= 5.0


def test_posterior_variance_at_planck_size_within_its_standard_error():
    """Full size (planck, L = 10, the bench's CG launch configuration): every one of the 4M entries
    of the 8-probe estimate within 7 standard errors of the exact diagonal (DCT closed form), and the
    RMS standardised error at the predicted scale."""
    from synth import make_config
    p = make_config("planck")[0]
    ctx, _ = make_ctx([p])
    s = 8
    var, rep = ctx.posterior_variance(s, seed=21, tol=1e-10)
    var = var.cpu().numpy().reshape(p.k, -1)
    d1, d2 = variance.dct_diag_moments(p.level, p.A, p.noise_prec, p.tau, p.kappa2)
    sig = np.sqrt((d2 - d1 ** 2) / s)
    z = np.abs(var - d1) / sig
    assert z.max() <= 7.0, z.max()
    assert 0.8 < np.sqrt(np.mean(z ** 2)) < 1.2


def test_posterior_variance_d2_prior_with_hits():
    """The paper's operator (D^2 prior, random hits): GPU estimate == oracle estimate, same probes."""
    ps = [make_patch(5, 9, 3, seed=570 + s, tau="loguniform", prior="d2", hits="random") for s in range(2)]
    ctx, _ = make_ctx(ps)
    var, rep = ctx.posterior_variance(4, seed=9, tol=TOL)
    var = var.cpu().numpy().reshape(2, -1)
    ref = variance.hutchinson([model.problem_system(p)[0] for p in ps], 3, ps[0].N, 4, seed=9, tol=TOL)
    assert np.abs(var - ref).max() <= 1e-8 * np.abs(ref).max()
