"""The seeded generator: determinism, shapes, draw ranges (BASELINE.json configs)."""

import numpy as np

from synth import CONFIGS, make_config, make_patch
from synth.problems import stack


def test_determinism_and_shapes():
    a = make_patch(4, 9, 3, seed=0)
    b = make_patch(4, 9, 3, seed=0)
    c = make_patch(4, 9, 3, seed=1)
    assert np.array_equal(a.Y, b.Y) and np.array_equal(a.A, b.A)
    assert not np.array_equal(a.Y, c.Y)
    assert a.Y.shape == (9, 16, 16) and a.S.shape == (3, 16, 16)
    assert np.all(a.A[:, 0] == 1.0) and np.all((a.A[:, 1:] >= 0.1) & (a.A[:, 1:] <= 2.0))
    s2 = 1 / a.noise_prec
    assert np.all((s2 >= 1e-2) & (s2 <= 1.0))
    assert list(a.tau) == [1.0, 10.0, 100.0] and a.kappa2 == 0.1


def test_config_recipes():
    assert [CONFIGS[c]["level"] for c in ("tiny", "medium", "planck", "fullsky", "stress")] == \
        [5, 8, 10, 10, 11]
    assert CONFIGS["fullsky"]["seeds"] == list(range(100, 112))
    p = make_patch(3, 9, 6, seed=3, tau="logspace", kappa2="loguniform")
    assert np.allclose(p.tau, np.logspace(0, 4, 6)) and 1e-3 <= p.kappa2 <= 1
    q = make_patch(3, 9, 4, seed=2, tau="loguniform")
    assert np.all((q.tau >= 1) & (q.tau <= 1e3))


def test_stack_layout():
    ps = make_config("tiny") + make_config("tiny")
    st = stack(ps)
    assert st["A"].shape == (2, 9, 3) and st["Y"].shape == (2, 9, 32, 32)
    assert st["hits"] is None and st["kappa2"].shape == (2,)
