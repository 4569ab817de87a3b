"""GPU parity of the block-Lanczos Sylvester solver (Alg. SylvSolver; SURVEY 8(f)
NEXT-1) through the C ABI (sylvester_lanczos_solve) against the oracle's step-by-step
implementation (oracle/lanczos.py) and the exact solutions.

Bar: relative 2-norm error <= 1e-8 against the oracle's iterate at tol 1e-10 and Lanczos step
counts within +-2 (reading R18); both within 1e-8 of the DCT-exact / dense solution.  The GPU
evaluates the same iteration in a different (exact-arithmetic-equivalent) order: one Gram
reduction per step, W recomputed instead of stored, gamma by block elimination (readings R29-R31).
"""

import json
import os

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from oracle import exact, lanczos, model
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

TOL = 1e-10
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "oracle_iterations.json")


def _np(t):
    return t.detach().cpu().numpy()


def _run(ps, cap=400, store=False, tol=TOL, max_iter=100000, **kw):
    ctx, Y = make_ctx(ps, lanczos_cap=cap, lanczos_store=store, **kw)
    mu, rep = ctx.lanczos(Y, tol=tol, max_iter=max_iter)
    return ctx, Y, _np(mu), rep


def _check(ps, its_tol=2, err_tol=1e-8, **kw):
    ctx, Y, mu, rep = _run(ps, **kw)
    assert rep["converged"], rep
    for i, p in enumerate(ps):
        ref = lanczos.problem_solve(p, tol=TOL)
        assert ref.converged
        assert rel(mu[i], ref.x) <= err_tol, (i, rel(mu[i], ref.x))
        assert abs(rep["iterations_per"][i] - ref.iterations) <= its_tol, (i, rep["iterations_per"][i], ref.iterations)
    return ctx, Y, mu, rep


def test_lanczos_tiny_vs_oracle_and_exact():
    ps = make_config("tiny")
    ctx, Y, mu, rep = _check(ps)
    assert rel(mu[0], exact.problem_dct_exact(ps[0])) <= 1e-8
    assert rep["rel_residual_true"] <= 1e-8
    assert rep["rel_residual"] <= TOL


def test_lanczos_medium_vs_oracle_and_exact():
    ps = make_config("medium")
    ctx, Y, mu, rep = _check(ps)
    assert rel(mu[0], exact.problem_dct_exact(ps[0])) <= 1e-8


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 8])
def test_lanczos_every_k_batched_faces(k):
    """Three faces with different parameters in one launch (per-face freeze), ragged 2^5 face
    (narrower than one 64-pixel tile), every K instantiation."""
    ps = [make_patch(5, 9, k, seed=60 + 7 * k + s, tau="loguniform") for s in range(3)]
    _check(ps)


@pytest.mark.parametrize("level", [6, 7])
def test_lanczos_hits(level):
    ps = [make_patch(level, 9, 3, seed=70 + s, tau="loguniform", hits="random") for s in range(2)]
    ctx, Y, mu, rep = _check(ps)
    for i, p in enumerate(ps):
        G, b = model.problem_system(p)
        r = G @ mu[i].reshape(-1) - b
        assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b)


def test_lanczos_store_equals_replay_bitwise():
    """HBM-resident basis + one assembly pass == the paper's second Lanczos pass, bit for bit."""
    ps = [make_patch(6, 9, 4, seed=80 + s, tau="loguniform") for s in range(3)]
    _, _, mu_r, rep_r = _run(ps, store=False)
    _, _, mu_s, rep_s = _run(ps, store=True, cap=200)
    assert rep_r["iterations_per"] == rep_s["iterations_per"]
    assert np.array_equal(mu_r, mu_s)


def test_lanczos_repeatable_bitwise():
    ps = [make_patch(7, 9, 4, seed=90, tau="loguniform")]
    ctx, Y = make_ctx(ps, lanczos_cap=300)
    a, _ = ctx.lanczos(Y, tol=TOL)
    a = _np(a)
    b, _ = ctx.lanczos(Y, tol=TOL)
    assert np.array_equal(a, _np(b))


def test_lanczos_max_iter_gives_galerkin_iterate():
    """Stopped at step m: mu = the Galerkin solution at step m (the oracle's x at max_iter)."""
    ps = [make_patch(6, 9, 3, seed=95, tau="loguniform")]
    for m in (1, 2, 5, 17):
        ctx, Y, mu, rep = _run(ps, max_iter=m)
        assert rep["status"] == 1 and rep["iterations"] == m, rep  # KCG_NOT_CONVERGED
        ref = lanczos.problem_solve(ps[0], tol=TOL, max_iter=m)
        assert rel(mu[0], ref.x) <= 1e-10, (m, rel(mu[0], ref.x))


def test_lanczos_cap_limits_steps():
    ps = [make_patch(6, 9, 3, seed=96, tau="loguniform")]
    ctx, Y, mu, rep = _run(ps, cap=7)
    assert rep["iterations"] == 7 and not rep["converged"]


def test_lanczos_zero_rhs():
    import torch
    ps = [make_patch(5, 9, 3, seed=97)]
    ctx, Y = make_ctx(ps, lanczos_cap=50)
    mu, rep = ctx.lanczos(torch.zeros_like(Y), tol=TOL)
    assert rep["converged"] and rep["iterations"] == 0
    assert float(mu.abs().max()) == 0.0


def test_lanczos_exhausted_krylov_space_is_exact():
    """k = 1 on a 2x2 face (N = 4): the Krylov space is exhausted after at most 4 steps, the
    projection is then exact (B = 0 to rounding); N = 1 after one step."""
    for level in (0, 1):
        p = make_patch(level, 3, 1, seed=98, tau="given", tau_values=[2.0])
        ctx, Y, mu, rep = _run([p], tol=1e-14)
        G, b = model.problem_system(p)
        assert rep["converged"], rep
        assert rel(mu[0], exact.dense_solve(G, b)) <= 1e-12


def test_lanczos_nested_layout_is_a_permutation():
    """NESTED (reading R1) input gathered into the kernels' row-major layout, the solution
    scattered back: the same solve permuted."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.problems import stack
    p = make_patch(6, 9, 3, seed=99, tau="loguniform", hits="random")
    ctx_r, Y = make_ctx([p], lanczos_cap=300)
    mu_r, rep_r = ctx_r.lanczos(Y, tol=TOL)
    st = stack([p])
    nest = lambda a: model.to_layout(p.level, a, "nested").reshape(np.shape(a))
    ctx_n = KronCG(p.level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                   hits=torch.from_numpy(nest(st["hits"])).cuda(), layout="nested", lanczos_cap=300)
    mu_n, rep_n = ctx_n.lanczos(torch.from_numpy(nest(st["Y"])).cuda(), tol=TOL)
    assert rep_n["iterations_per"] == rep_r["iterations_per"]
    assert np.array_equal(_np(mu_n), nest(_np(mu_r)))


def test_lanczos_planck_vs_exact():
    """planck (L = 10, k = 4, one face) at the size bench.py times: DCT-exact solution and the
    oracle's step count (tests/golden, written by scripts/oracle_lanczos_iterations.py)."""
    ps = make_config("planck")
    ctx, Y, mu, rep = _run(ps, cap=300, store=True)
    assert rep["converged"]
    assert rel(mu[0], exact.problem_dct_exact(ps[0])) <= 1e-8
    gold = json.load(open(GOLDEN))["planck"].get("lanczos_iterations")
    if gold:
        assert abs(rep["iterations_per"][0] - gold[0]) <= 2


def test_lanczos_fullsky_sample_faces_vs_exact():
    """Four of the twelve fullsky faces batched (per-face parameters, literal reading R20)."""
    ps = make_config("fullsky", patches=[0, 3, 7, 11])
    ctx, Y, mu, rep = _run(ps, cap=400, store=False)
    assert rep["converged"]
    gold = json.load(open(GOLDEN))["fullsky"].get("lanczos_iterations")
    for i, (p, fi) in enumerate(zip(ps, [0, 3, 7, 11])):
        assert rel(mu[i], exact.problem_dct_exact(p)) <= 1e-8
        if gold:
            assert abs(rep["iterations_per"][i] - gold[fi]) <= 2


@pytest.mark.parametrize("k,hits", [(1, None), (2, "random"), (3, None), (4, "random")])
def test_lanczos_d2_prior_vs_oracle(k, hits):
    """The paper's operator N_h^{-1} D^2 (+ kappa2), radius 2: halo-4 boxes, D V formed in shared
    memory on the tile + 3 ring (step A) and + 1 ring (step B)."""
    ps = [make_patch(6, 9, k, seed=300 + 11 * k + s, tau="loguniform", prior="d2", hits=hits) for s in range(2)]
    _check(ps, prior="d2")


def test_lanczos_d2_planck_vs_exact():
    ps = make_config("planck", prior="d2")
    ctx, Y, mu, rep = _run(ps, cap=300, store=True, prior="d2")
    assert rep["converged"]
    assert rel(mu[0], exact.problem_dct_exact(ps[0])) <= 1e-8


def test_lanczos_host_entry_point_matches_device():
    """sylvester_lanczos_solve_host: Y from host memory in, mu to host memory out (copies timed)."""
    import torch
    ps = [make_patch(6, 9, 3, seed=610 + s, tau="loguniform") for s in range(2)]
    ctx, Y = make_ctx(ps, lanczos_cap=200, host_staging=True)
    mu_d, rep_d = ctx.lanczos(Y, tol=TOL)
    mu_h, rep_h = ctx.solve_host(Y.cpu().pin_memory(), tol=TOL, route="lanczos")
    assert rep_h["iterations_per"] == rep_d["iterations_per"]
    assert np.array_equal(mu_h.numpy(), _np(mu_d))
    assert rep_h["wall_time_s"] >= rep_h["loop_time_s"] > 0


def test_lanczos_configuration_errors():
    from paper_2204_08057_b200.kroncg import KcgError, KCG_E_CONFIG
    ps = [make_patch(5, 9, 3, seed=620)]
    ctx, Y = make_ctx(ps)                       # no lanczos_cap: route not provisioned
    with pytest.raises(KcgError) as e:
        ctx.lanczos(Y, tol=TOL)
    assert e.value.status == KCG_E_CONFIG
    ps5 = [make_patch(5, 9, 5, seed=621, prior="d2")]
    with pytest.raises(KcgError) as e:          # D^2 block Lanczos is built for k <= 4
        make_ctx(ps5, lanczos_cap=50)
    assert e.value.status == KCG_E_CONFIG


def test_max_level_all_routes_vs_exact():
    """The largest face the ABI accepts (level 12: 4096 x 4096, 16.8M pixels): Kronecker CG, the
    Sylvester route and block Lanczos (paper's two-pass mode) against the DCT-exact solution."""
    p = make_patch(12, 4, 2, seed=700, tau="loguniform")
    ex = exact.problem_dct_exact(p)
    ctx, Y = make_ctx([p], lanczos_cap=400)
    for name, fn in (("kron", ctx.solve), ("sylvester", ctx.sylvester), ("lanczos", ctx.lanczos)):
        mu, rep = fn(Y, tol=TOL)
        assert rep["converged"], (name, rep["status_name"])
        assert rel(_np(mu)[0], ex) <= 1e-8, (name, rel(_np(mu)[0], ex))


def test_lanczos_nonfinite_and_rank_deficient_inputs():
    """NaN in the data -> KCG_E_NONFINITE; a rank-deficient starting block Y^ (identical maps make
    Y T A P^{-1} rank one for k = 3) -> the Cholesky QR of B_0 breaks down: KCG_E_BREAKDOWN."""
    from paper_2204_08057_b200.kroncg import KcgError, KCG_E_NONFINITE, KCG_E_BREAKDOWN
    ps = [make_patch(4, 9, 3, seed=630)]
    ctx, Y = make_ctx(ps, lanczos_cap=50)
    Yn = Y.clone()
    Yn[0, 2, 3, 3] = float("nan")
    with pytest.raises(KcgError) as e:
        ctx.lanczos(Yn, tol=TOL)
    assert e.value.status == KCG_E_NONFINITE
    Yr = Y.clone()
    Yr[0] = Y[0, :1].expand_as(Y[0])                  # every map the same: Y has rank one
    with pytest.raises(KcgError) as e:
        ctx.lanczos(Yr.contiguous(), tol=TOL)
    assert e.value.status == KCG_E_BREAKDOWN


def test_lanczos_batch_composition_changes_only_rounding():
    """Sharding faces across ranks changes the per-CTA Gram partial grouping (chunks follow the batch),
    so a face solved alone and inside a batch agree to rounding, with the same step count."""
    ps = [make_patch(7, 9, 4, seed=640 + s, tau="loguniform") for s in range(3)]
    _, _, mu_b, rep_b = _run(ps, cap=300)
    for i, p in enumerate(ps):
        _, _, mu_1, rep_1 = _run([p], cap=300)
        assert rep_1["iterations_per"][0] == rep_b["iterations_per"][i]
        assert rel(mu_1[0], mu_b[i]) <= 1e-12
