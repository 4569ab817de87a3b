"""GPU tests of the C ABI's argument contract (include/kroncg.h "Errors"): hit counts validated on the
device at create, host-buffer shape/dtype checks in the binding, the level-0 block-Jacobi block, and
the per-patch iteration counts of posterior_variance."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from oracle import cg, model
from synth import make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
TOL = 1e-10


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf")])
def test_nonpositive_hits_rejected(bad):
    import torch
    from paper_2204_08057_b200.kroncg import KcgError, KronCG
    from synth.problems import stack
    ps = [make_patch(4, 9, 3, seed=1, hits="random"), make_patch(4, 9, 3, seed=2, hits="random")]
    st = stack(ps)
    h = torch.from_numpy(st["hits"]).cuda()
    h[1, 7, 3] = bad
    with pytest.raises(KcgError) as e:
        KronCG(4, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=h)
    assert e.value.status == 2 and "hits" in str(e.value)


def test_slab_hits_ghost_rows_may_be_zero_but_own_rows_not():
    import torch
    from paper_2204_08057_b200.kroncg import KcgError, KronCGSlab
    from synth.problems import stack
    p = make_patch(5, 9, 3, seed=3, hits="random")
    st = stack([p])
    h = torch.from_numpy(st["hits"]).cuda()
    KronCGSlab(5, st["A"], st["noise_prec"], st["tau"], st["kappa2"], 2, emulate=True, hits=h)  # face-edge ghosts = 0
    h[0, 20, 5] = 0.0
    with pytest.raises(KcgError) as e:
        KronCGSlab(5, st["A"], st["noise_prec"], st["tau"], st["kappa2"], 2, emulate=True, hits=h)
    assert e.value.status == 2


def test_solve_host_checks_buffers():
    import torch
    ctx, Y = make_ctx([make_patch(3, 9, 2, seed=4)], host_staging=True)
    Yh = Y.cpu()
    with pytest.raises(ValueError):
        ctx.solve_host(Yh.float())
    with pytest.raises(ValueError):
        ctx.solve_host(Yh[..., :4])
    with pytest.raises(ValueError):
        ctx.solve_host(Yh.transpose(-1, -2))
    with pytest.raises(ValueError):
        ctx.solve_host(Yh, mu=torch.empty((1, 2, 8, 4), dtype=torch.float64))
    mu, rep = ctx.solve_host(Yh.numpy(), tol=TOL)
    assert rep["converged"]


@pytest.mark.parametrize("k,hits", [(1, None), (3, None), (4, "random")])
def test_block_jacobi_level0(k, hits):
    """Level 0: one pixel, degree 0 -- the preconditioner is the exact inverse of the k x k G, so PCG
    stops after one iteration (the degree-0 block is built on the host, kinv_slot(0))."""
    ps = [make_patch(0, 9, k, seed=30 + s, tau="loguniform", hits=hits) for s in range(2)]
    ctx, Y = make_ctx(ps, precond="block_jacobi")
    mu, rep = ctx.solve(Y, tol=TOL)
    mu = mu.cpu().numpy()
    assert rep["converged"]
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        x = np.linalg.solve(G.toarray(), b)
        assert rel(mu[i], x) <= 1e-12
        assert rep["iterations_per"][i] == 1


def test_posterior_variance_reports_iterations_per_patch():
    ps = [make_patch(5, 9, 3, seed=40 + s, tau="loguniform") for s in range(3)]
    ctx, _ = make_ctx(ps)
    _, rep = ctx.posterior_variance(3, seed=5, tol=TOL)
    its = rep["iterations_per"]
    assert len(its) == 3 and all(v > 0 for v in its) and max(its) == rep["iterations"]
    # each entry is the largest count over the probes: at least one probe's own oracle count
    from oracle import variance
    for i, p in enumerate(ps):
        G, _ = model.problem_system(p)
        counts = []
        for q in range(3):
            z = variance.rademacher(5, q, len(ps), p.k, p.N)[i].reshape(-1)
            counts.append(cg.cg_hs(G, z, tol=TOL).iterations)
        assert abs(its[i] - max(counts)) <= 2, (its[i], counts)


def test_misaligned_mu_rejected():
    """Device solutions are stored as pixel pairs (double2): a mu that is not 16-byte aligned is an
    argument error (kroncg.h), never a misaligned store."""
    import torch
    from gpu_util import make_ctx
    from paper_2204_08057_b200.kroncg import KcgError
    from synth import make_patch
    ps = [make_patch(4, 9, 3, seed=1)]
    ctx, Y = make_ctx(ps)
    buf = torch.zeros(ctx.shape_mu[0] * 3 * 16 * 16 + 1, dtype=torch.float64, device="cuda")
    mu = buf[1:].view(ctx.shape_mu)  # offset by one double: 8-byte aligned only
    for fn in (ctx.solve, ctx.sylvester, ctx.kohler):
        with pytest.raises(KcgError) as e:
            fn(Y, mu)
        assert e.value.status == 2


@pytest.mark.parametrize("nb", [1, 2, 5])
def test_solve_host_many_pipeline(nb):
    """kron_cg_solve_host_many (two staging pairs, copies queued after each solve's kernels): batch i's
    mu from Ys[i] equals the device-resident solve of the same Y bit for bit (the same kernels on the
    same data), with the same iteration counts; every batch has its own input, output and report; the
    first batch is also checked against the oracle."""
    import torch
    ps = [make_patch(5, 9, 3, seed=60 + s, tau="loguniform") for s in range(3)]
    ctx, Y = make_ctx(ps, host_staging=2)
    Ys = [(Y.cpu() * (1.0 + 0.25 * i)).pin_memory() for i in range(nb)]
    mus = [torch.full(tuple(ctx.shape_mu), float("nan"), dtype=torch.float64).pin_memory() for _ in range(nb)]
    reps = ctx.solve_host_many(Ys, mus, tol=TOL)
    assert len(reps) == nb
    for i in range(nb):
        mu_d, rep_d = ctx.solve(Ys[i].cuda(), tol=TOL)
        assert reps[i]["converged"] and reps[i]["iterations_per"] == rep_d["iterations_per"], (i, reps[i], rep_d)
        assert torch.equal(mus[i], mu_d.cpu()), i
    for j, p in enumerate(ps):
        G, b = model.problem_system(p)
        ref = cg.cg_hs(G, b, tol=TOL)
        assert rel(mus[0][j].numpy(), ref.x) <= 1e-8
        assert abs(reps[0]["iterations_per"][j] - ref.iterations) <= 2
