"""GPU parity of the row-slab decomposition: every face split into G row slabs,
all G ranks emulated on this GPU in ONE cooperative launch (one CTA group per rank; halo rows
stored into the neighbours' ghost rows, per-iteration cross-rank sums through slots + flags --
the same device code a one-process-per-GPU run executes).  Compared with the oracle and with the
unsplit solve."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from oracle import cg, exact, model, sylvester
from synth import make_config, make_patch
from synth.problems import stack

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

TOL = 1e-10


def _slab_ctx(ps, G, **kw):
    import torch
    from paper_2204_08057_b200 import build
    build.build()
    from paper_2204_08057_b200.kroncg import KronCGSlab, split_rows
    st = stack(ps)
    hits = torch.from_numpy(st["hits"]).cuda() if st["hits"] is not None else None
    ctx = KronCGSlab(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], G, emulate=True,
                     hits=hits, **kw)
    Y = split_rows(torch.from_numpy(st["Y"]), G).cuda()
    return ctx, Y


def _join(mu):
    from paper_2204_08057_b200.kroncg import join_rows
    return join_rows(mu).cpu().numpy()


@pytest.mark.parametrize("level,k,G,hits", [(3, 3, 2, None), (5, 3, 4, None), (5, 4, 8, "random"),
                                            (6, 2, 2, "random"), (7, 4, 4, None), (6, 6, 8, None),
                                            (4, 1, 4, None)])
def test_slab_kron_vs_oracle_and_unsplit(level, k, G, hits):
    ps = [make_patch(level, 9, k, seed=130 + s, tau="loguniform", hits=hits) for s in range(2)]
    ctx, Y = _slab_ctx(ps, G)
    mu, rep = ctx.solve(Y, tol=TOL)
    mu = _join(mu)
    assert rep["converged"], rep
    c1, Y1 = make_ctx(ps)
    mu1, rep1 = c1.solve(Y1, tol=TOL)
    mu1 = mu1.cpu().numpy()
    for i, p in enumerate(ps):
        G_, b = model.problem_system(p)
        ref = cg.cg_hs(G_, b, tol=TOL)
        assert rel(mu[i], ref.x) <= 1e-8, (i, rel(mu[i], ref.x))
        assert abs(rep["iterations_per"][i] - ref.iterations) <= 2
        assert abs(rep["iterations_per"][i] - rep1["iterations_per"][i]) <= 1
        assert rel(mu[i], mu1[i]) <= 1e-9
    assert rep["rel_residual_true"] <= 5 * TOL


def test_slab_medium_sylvester_and_pcg():
    ps = make_config("medium")
    ctx, Y = _slab_ctx(ps, 4)
    mu, rep = ctx.sylvester(Y, tol=TOL)
    ref = sylvester.problem_solve(ps[0], tol=TOL)
    assert rel(_join(mu)[0], ref.x) <= 1e-8
    assert all(abs(a - b) <= 2 for a, b in zip(rep["iterations_per"], ref.iterations)), (rep["iterations_per"], ref.iterations)
    ctx2, Y2 = _slab_ctx(ps, 4, precond="block_jacobi")
    mu2, rep2 = ctx2.solve(Y2, tol=TOL)
    G_, b = model.problem_system(ps[0])
    K = cg.block_jacobi_precond(ps[0].level, ps[0].A, ps[0].noise_prec, ps[0].tau, ps[0].kappa2)
    ref2 = cg.cg_hs(G_, b, tol=TOL, precond=K)
    assert rel(_join(mu2)[0], ref2.x) <= 1e-8 and abs(rep2["iterations"] - ref2.iterations) <= 2


def test_slab_apply_matches_unsplit():
    import torch
    from paper_2204_08057_b200.kroncg import split_rows
    ps = [make_patch(6, 9, 4, seed=140 + s, tau="loguniform", hits="random") for s in range(2)]
    ctx, _ = _slab_ctx(ps, 8)
    c1, _ = make_ctx(ps)
    x = torch.randn((2, 4, 64, 64), dtype=torch.float64, device="cuda")
    y1 = c1.apply(x).cpu().numpy()
    ys = _join(ctx.apply(split_rows(x, 8)))
    assert np.allclose(ys, y1, rtol=1e-13, atol=1e-13 * np.abs(y1).max())


def test_slab_planck_full_size_vs_exact():
    p = make_config("planck")[0]
    ctx, Y = _slab_ctx([p], 8)
    mu, rep = ctx.solve(Y, tol=TOL)
    assert rep["converged"] and rep["rel_residual_true"] <= 5 * TOL
    assert rel(_join(mu)[0], exact.problem_dct_exact(p)) <= 1e-8


def test_slab_deterministic_and_host_entry():
    import torch
    ps = [make_patch(7, 9, 3, seed=150, tau="loguniform")]
    ctx, Y = _slab_ctx(ps, 4, host_staging=True)
    m1, r1 = ctx.solve(Y, tol=TOL)
    m2, r2 = ctx.solve(Y, tol=TOL)
    assert torch.equal(m1, m2) and r1["iterations"] == r2["iterations"]
    m3, r3 = ctx.solve_host(Y.cpu().pin_memory(), tol=TOL)
    assert np.array_equal(m1.cpu().numpy(), m3.numpy()) and r3["iterations"] == r1["iterations"]


def test_slab_rejects_bad_split():
    from paper_2204_08057_b200.kroncg import KcgError
    with pytest.raises((ValueError, KcgError)):
        _slab_ctx([make_patch(3, 9, 2, seed=1)], 4)   # 8 rows / 4 ranks = 2-row slabs < 4
