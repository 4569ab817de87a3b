"""The paper's own workload: App. B physics for A, the printed T, phi = 1,
the D^2 prior with kappa2 = 0, non-uniform hits, HEALPix NESTED order.

Pins: the App. B formulas reproduce the printed 9 x 4 mixing matrix (golden fixture
tests/golden/paper_appB.json, copied from the paper), and the oracle solves the paper system
exactly (direct sparse solve) in a handful of CG iterations (clustered spectrum)."""

import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as ssl

from oracle import cg, lanczos, model, sylvester
from synth.physics import PLANCK_T, make_paper_patch, planck_mixing

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_appB.json")))


def test_appB_formulas_reproduce_the_printed_mixing_matrix():
    A = planck_mixing()
    P = np.array(GOLD["A"])
    assert A.shape == P.shape == (9, 4)
    assert np.all(A[:, 0] == 1.0)                       # CMB column
    assert np.abs(A - P).max() <= 5e-3                  # three printed decimals (+ rounding of h, k_B)
    assert np.all(np.abs(A - P) <= 5e-4 * np.abs(P) + 1.5e-3)
    # at the reference frequency every foreground equals c(nu0)
    assert np.allclose(A[3, 1:], A[3, 1])


def test_printed_noise_precisions():
    assert list(PLANCK_T) == GOLD["T"]


def test_paper_patch_shapes_and_draw_order():
    p = make_paper_patch(3, seed=5)
    assert p.Y.shape == (9, 8, 8) and p.S.shape == (4, 8, 8) and p.hits.shape == (8, 8)
    assert p.prior == "d2" and p.kappa2 == 0.0 and np.all(p.tau == 1.0)
    q = make_paper_patch(3, seed=5)
    assert np.array_equal(p.Y, q.Y) and np.array_equal(p.hits, q.hits)
    assert set(np.unique(p.hits)) <= {1.0, 2.0, 3.0, 4.0}


@pytest.mark.parametrize("layout", ["row", "nested"])
def test_paper_system_oracle_routes_agree_with_the_direct_solve(layout):
    """kappa2 = 0: Q0 = D^2 is singular (constants) but G = M (x) N_h + I (x) D^2 is SPD
    because M = A^T T A is; CG, the Sylvester route and block Lanczos all reach G^{-1} b."""
    p = make_paper_patch(4, seed=11)
    G, b = model.problem_system(p, layout=layout)
    ref = ssl.spsolve(G.tocsc(), b)
    r = cg.cg_hs(G, b, tol=1e-10)
    assert r.converged and r.iterations < 200
    # cond(G) ~ 2e4 here (T ~ 1e6..3e7 against D^2 <= 64 hits): error <= cond * tol
    assert np.linalg.norm(G @ r.x - b) <= 2e-10 * np.linalg.norm(b)
    assert np.linalg.norm(r.x - ref) <= 1e-5 * np.linalg.norm(ref)
    if layout == "row":
        s = sylvester.problem_solve(p, tol=1e-10)
        assert np.linalg.norm(s.x - ref) <= 1e-8 * np.linalg.norm(ref)
        lz = lanczos.problem_solve(p, tol=1e-10)
        assert lz.converged
        assert np.linalg.norm(lz.x - ref) <= 1e-8 * np.linalg.norm(ref)
        # the shifts rho_j of S^ = A^T T A (P = I) dwarf D^2: the shifted systems are nearly
        # identities and the Sylvester routes converge in a few steps
        assert max(s.iterations) < 20 and lz.iterations < 10


def test_synth_nested_order_is_the_healpix_nested_numbering():
    """synth's input reordering (bench.py's paper leg) == the oracle's NESTED numbering (reading R1)."""
    from synth.physics import nested_order
    a = np.random.default_rng(0).standard_normal((2, 3, 16, 16))
    assert np.array_equal(nested_order(a), model.to_layout(4, a, "nested").reshape(a.shape))
