"""GPU parity of the warm start (kron_cg_solve_x0, reading R37; SURVEY 5 "warm start"): r_0 = b - G x_0,
stopping rule relative to ||b|| -- against the oracle's textbook CG started from the same x_0
(oracle/cg.py cg_hs(x0=...)), element by element at 1e-8 and iteration counts within the oracle's
rounding envelope (reading R34)."""

import numpy as np
import pytest
import scipy.sparse.linalg as ssl

from gpu_util import have_gpu, make_ctx, oracle_count_envelope, rel
from oracle import cg, exact, model
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
TOL = 1e-10


def _guess(p, scale, seed):
    """x_0 = the exact solution plus a seeded perturbation of relative size `scale` (a neighbouring
    parameter set's solution, say): [k][side][side]."""
    G, b = model.problem_system(p)
    xs = ssl.spsolve(G.tocsc(), b)
    rng = np.random.default_rng(seed)
    return (xs + scale * np.linalg.norm(xs) / np.sqrt(xs.size) * rng.standard_normal(xs.size)).reshape(
        p.k, 1 << p.level, 1 << p.level)


def _check(ps, x0s, precond=None, **kw):
    import torch
    ctx, Y = make_ctx(ps, precond=precond or "none", **kw)
    x0 = torch.from_numpy(np.stack(x0s)).cuda()
    mu, rep = ctx.solve(Y, tol=TOL, x0=x0)
    mu = mu.cpu().numpy()
    assert rep["converged"], rep["status_name"]
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2, p.hits,
                                    prior=p.prior) if precond else None
        lo, hi, ref = oracle_count_envelope(cg.cg_hs, G, b, tol=TOL, precond=K, x0=x0s[i].reshape(-1))
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        assert lo - 2 <= rep["iterations_per"][i] <= hi + 2, (i, rep["iterations_per"][i], lo, hi)
    assert rep["rel_residual_true"] <= 5 * TOL
    return ctx, Y, mu, rep


@pytest.mark.parametrize("level,k,hits,prior", [(2, 3, None, "laplacian"), (5, 4, "random", "laplacian"),
                                                (6, 2, None, "d2"), (7, 3, "random", "laplacian"),
                                                (8, 4, None, "laplacian")])
def test_warm_start_vs_oracle(level, k, hits, prior):
    ps = [make_patch(level, 9, k, seed=830 + s, tau="loguniform", hits=hits, prior=prior) for s in range(2)]
    _check(ps, [_guess(p, 1e-3, 7 + i) for i, p in enumerate(ps)])


def test_warm_start_block_jacobi():
    ps = [make_patch(6, 9, 3, seed=840 + s, tau="loguniform", hits="random") for s in range(2)]
    _check(ps, [_guess(p, 1e-2, 9 + i) for i, p in enumerate(ps)], precond="block_jacobi")


def test_warm_start_saves_iterations_and_edge_cases():
    import torch
    ps = make_config("medium")
    ctx, Y = make_ctx(ps)
    _, cold = ctx.solve(Y, tol=TOL)
    x0 = torch.from_numpy(np.stack([_guess(ps[0], 1e-4, 1)])).cuda()
    mu, warm = ctx.solve(Y, tol=TOL, x0=x0)
    assert warm["converged"] and warm["iterations"] < cold["iterations"]
    assert rel(mu.cpu().numpy()[0], exact.problem_dct_exact(ps[0])) <= 1e-8
    # x0 = 0: the cold start's iterates (r_0 = b - G 0 = b exactly); the stopping threshold uses
    # ||b|| from the residual kernel, so only the count at the boundary could move
    m0, r0 = ctx.solve(Y, tol=TOL, x0=torch.zeros_like(x0))
    mc, _ = ctx.solve(Y, tol=TOL)
    assert abs(r0["iterations"] - cold["iterations"]) <= 1 and rel(m0.cpu().numpy(), mc.cpu().numpy()) <= 1e-12
    # x0 = a converged solution: 0 iterations, x returned unchanged; x0 may alias mu
    xs = mc.clone()
    m1, r1 = ctx.solve(Y, mu=xs, tol=1e-6, x0=xs)
    assert r1["iterations"] == 0 and r1["converged"] and torch.equal(m1, mc)
    # b = 0: the solution is 0 (the rule falls back to ||r_0||)
    mz, rz = ctx.solve(torch.zeros_like(Y), tol=1e-8, x0=x0)
    assert rz["converged"] and mz.abs().max().item() <= 1e-6 * x0.abs().max().item()


def test_warm_start_tiny_resident_and_nested():
    """The single-CTA resident kernel (tiny faces) and the NESTED layout take x_0 too."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.problems import stack
    ps = make_config("tiny")
    ctx, Y = make_ctx(ps)
    assert ctx.launch_config()["resident_kron"] == 1
    x0 = _guess(ps[0], 1e-3, 5)
    _check(ps, [x0])
    # NESTED: x0 and mu in the user's (nested) order
    st = stack(ps)
    L = ps[0].level
    nest = lambda a: model.to_layout(L, a, "nested").reshape(np.shape(a))
    cn = KronCG(L, st["A"], st["noise_prec"], st["tau"], st["kappa2"], layout="nested")
    mu, rep = cn.solve(torch.from_numpy(nest(st["Y"])).cuda(), tol=TOL,
                       x0=torch.from_numpy(nest(x0[None])).cuda())
    G, b = model.problem_system(ps[0], layout="nested")
    ref = cg.cg_hs(G, b, tol=TOL, x0=nest(x0[None]).reshape(-1))
    assert rel(mu.cpu().numpy()[0], ref.x) <= 1e-8 and abs(rep["iterations"] - ref.iterations) <= 2


def test_warm_start_rejected_configs():
    import torch
    from paper_2204_08057_b200.kroncg import KcgError
    ps = [make_patch(4, 9, 3, seed=1)]
    ctx, Y = make_ctx(ps, cg_variant="hs")
    with pytest.raises(KcgError) as e:
        ctx.solve(Y, tol=TOL, x0=torch.zeros((1, 3, 16, 16), dtype=torch.float64, device="cuda"))
    assert e.value.status == 4
