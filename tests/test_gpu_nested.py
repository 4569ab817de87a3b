"""GPU parity of the NESTED pixel layout (reading R1; SURVEY 8(a) a2's NESTED -> row-major gather):
data maps, hits and solutions in HEALPix NESTED order inside each face, against the oracle system
assembled directly in NESTED numbering."""

import numpy as np
import pytest

from gpu_util import have_gpu, rel
from oracle import cg, grid, model, sylvester
from synth import make_config, make_patch
from synth.problems import stack

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

TOL = 1e-10


def _nested(level, a):
    """[..][side][side] row-major maps -> the same shape holding NESTED-ordered flat vectors."""
    return model.to_layout(level, a, "nested").reshape(np.shape(a))


def _ctx(ps, **kw):
    import torch
    from paper_2204_08057_b200 import build
    build.build()
    from paper_2204_08057_b200.kroncg import KronCG
    st = stack(ps)
    L = ps[0].level
    hits = torch.from_numpy(_nested(L, st["hits"])).cuda() if st["hits"] is not None else None
    ctx = KronCG(L, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=hits, layout="nested", **kw)
    return ctx, torch.from_numpy(_nested(L, st["Y"])).cuda()


@pytest.mark.parametrize("level,k,hits", [(0, 1, None), (3, 3, "random"), (5, 4, None), (7, 2, "random")])
def test_nested_kron_vs_oracle(level, k, hits):
    ps = [make_patch(level, 9, k, seed=160 + s, tau="loguniform", hits=hits) for s in range(2)]
    ctx, Y = _ctx(ps)
    mu, rep = ctx.solve(Y, tol=TOL)
    mu = mu.cpu().numpy()
    for i, p in enumerate(ps):
        G, b = model.problem_system(p, layout="nested")
        ref = cg.cg_hs(G, b, tol=TOL)
        assert rel(mu[i], ref.x) <= 1e-8
        assert abs(rep["iterations_per"][i] - ref.iterations) <= 2
    assert rep["rel_residual_true"] <= 5 * TOL


def test_nested_apply_rhs_sylvester_pcg():
    import torch
    ps = make_config("medium")
    p = ps[0]
    ctx, Y = _ctx(ps)
    G, b = model.problem_system(p, layout="nested")
    x = np.random.default_rng(0).standard_normal((1, p.k, p.side, p.side))
    y = ctx.apply(torch.from_numpy(x).cuda()).cpu().numpy().reshape(-1)
    ref = G @ x.reshape(-1)
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    bb = ctx.rhs(Y).cpu().numpy().reshape(-1)
    assert np.allclose(bb, b, rtol=1e-13, atol=1e-13 * np.abs(b).max())
    mu, rep = ctx.sylvester(Y, tol=TOL)
    sref = sylvester.problem_solve(p, tol=TOL)   # row-major oracle, compared after permuting
    perm = grid.pixel_index(p.level, "nested").reshape(-1)
    xr = sref.x.reshape(p.k, -1)
    xn = np.empty_like(xr)
    xn[:, perm] = xr
    assert rel(mu.cpu().numpy().reshape(-1), xn.reshape(-1)) <= 1e-8
    c2, Y2 = _ctx(ps, precond="block_jacobi")
    mu2, rep2 = c2.solve(Y2, tol=TOL)
    K = cg.block_jacobi_precond(p.level, p.A, p.noise_prec, p.tau, p.kappa2)
    ref2 = cg.cg_hs(*model.problem_system(p), tol=TOL, precond=K)   # row-major PCG, permuted
    xr2 = ref2.x.reshape(p.k, -1)
    xn2 = np.empty_like(xr2)
    xn2[:, perm] = xr2
    assert rel(mu2.cpu().numpy().reshape(-1), xn2.reshape(-1)) <= 1e-8
    assert abs(rep2["iterations"] - ref2.iterations) <= 2


def test_nested_slab_rejected():
    import torch
    from paper_2204_08057_b200.kroncg import KcgError, KronCGSlab, kcg_desc
    p = make_patch(5, 9, 2, seed=1)
    st = stack([p])
    # the Python slab wrapper is row-major only; the C ABI refuses the combination
    from paper_2204_08057_b200 import kroncg as kc
    import ctypes as C
    d = kcg_desc(5, 9, 2, 1, kc.KCG_PRIOR_LAPLACIAN, kc.KCG_LAYOUT_NESTED, kc.KCG_PRECOND_NONE, 0, 0)
    assert kc.kron_cg_workspace_size_slab(C.byref(d), 2) > 0
    ws = [torch.empty(kc.kron_cg_workspace_size_slab(C.byref(d), 2), dtype=torch.uint8, device="cuda") for _ in range(2)]
    sl = kc.kcg_slab()
    sl.nranks, sl.rank0, sl.nlocal = 2, 0, 2
    for r in range(2):
        sl.peer_ws[r] = ws[r].data_ptr()
    ctx = kc._ctxp()
    stt = kc.kron_cg_create_slab(C.byref(d), C.byref(sl), st["A"].ctypes.data, st["noise_prec"].ctypes.data,
                                 st["tau"].ctypes.data, st["kappa2"].ctypes.data, None, ws[0].numel(), None,
                                 C.byref(ctx))
    assert stt == kc.KCG_E_CONFIG
    kc.kron_cg_destroy(ctx)
