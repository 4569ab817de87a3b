"""GPU property tests at full size (SURVEY 4 "Kernel unit tests" / "Property tests"): closed forms
that hold at any level, so the CUDA path is checked at the bench's sizes without the oracle.

* DCT eigen-modes: with v_ab(y, x) = u_a(y) u_b(x) (orthonormal 2-D DCT-II basis) and hits = 1,
  G (v_ab (x) c) = v_ab (x) (M + lam_ab P) c,  lam_ab = kappa2 + l_ab (Laplacian) or l_ab^2 + kappa2
  (D^2), l_ab = (2 - 2 cos(pi a / s)) + (2 - 2 cos(pi b / s))  (the free-boundary grid spectrum).
* A single-mode right-hand side spans a k-dimensional invariant subspace: CG converges in <= k
  iterations (+1 for rounding) to v_ab (x) (M + lam_ab P)^{-1} c.
* Linearity of the solve in b (to the CG tolerance)."""

import numpy as np
import pytest

from gpu_util import have_gpu, make_ctx, rel
from synth import make_config, make_patch

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]


def _mode(s, a, b):
    def u(i):
        y = np.arange(s) + 0.5
        return (np.sqrt(1.0 / s) if i == 0 else np.sqrt(2.0 / s)) * np.cos(np.pi * i * y / s)
    return np.outer(u(a), u(b))


def _lam(s, a, b, kappa2, prior):
    l = (2 - 2 * np.cos(np.pi * a / s)) + (2 - 2 * np.cos(np.pi * b / s))
    return kappa2 + (l if prior == "laplacian" else l * l)


def _K(p, a, b):
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    return M + _lam(p.side, a, b, p.kappa2, p.prior) * np.diag(p.tau)


@pytest.mark.parametrize("prior", ["laplacian", "d2"])
def test_apply_on_dct_modes_at_planck_size(prior):
    import torch
    p = make_config("planck", prior=prior)[0]
    ctx, _ = make_ctx([p])
    s = p.side
    rng = np.random.default_rng(3)
    for a, b in [(0, 0), (1, 0), (5, 700), (1023, 1023), (512, 3)]:
        c = rng.standard_normal(p.k)
        v = _mode(s, a, b)
        x = np.einsum("c,yx->cyx", c, v)[None]
        y = ctx.apply(torch.from_numpy(x).cuda()).cpu().numpy()[0]
        ref = np.einsum("c,yx->cyx", _K(p, a, b) @ c, v)
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max(), (prior, a, b)


def test_single_mode_rhs_converges_in_k_iterations():
    import torch
    p = make_config("planck")[0]
    ctx, _ = make_ctx([p])
    s = p.side
    rng = np.random.default_rng(4)
    for a, b in [(2, 9), (300, 17)]:
        c = rng.standard_normal(p.k)
        v = _mode(s, a, b)
        bvec = np.einsum("c,yx->cyx", c, v)[None]
        x, rep = ctx.solve_b(torch.from_numpy(bvec).cuda(), tol=1e-12)
        assert rep["converged"] and rep["iterations"] <= p.k + 1, rep["iterations"]
        ref = np.einsum("c,yx->cyx", np.linalg.solve(_K(p, a, b), c), v)
        assert rel(x.cpu().numpy()[0], ref) <= 1e-10


def test_solve_is_linear_in_b():
    import torch
    p = make_patch(8, 9, 3, seed=900, tau="loguniform")
    ctx, _ = make_ctx([p])
    rng = np.random.default_rng(5)
    b1, b2 = rng.standard_normal((2, 1, 3, 256, 256))
    al, be = 0.7, -2.3
    x1, _ = ctx.solve_b(torch.from_numpy(b1).cuda(), tol=1e-12)
    x2, _ = ctx.solve_b(torch.from_numpy(b2).cuda(), tol=1e-12)
    x3, _ = ctx.solve_b(torch.from_numpy(al * b1 + be * b2).cuda(), tol=1e-12)
    lhs = x3.cpu().numpy()
    rhs = al * x1.cpu().numpy() + be * x2.cpu().numpy()
    assert rel(lhs, rhs) <= 1e-9
