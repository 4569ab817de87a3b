"""Pins for oracle.grid: SPEC worked examples, closed forms and the textbook grid spectrum."""

import json
import os

import numpy as np
import pytest

from oracle import grid, exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_neighbors_spec_examples():
    g = _gold("spec_grid_examples.json")
    for ex in g["neighbors"]:
        assert grid.neighbors(ex["level"], ex["j"]) == ex["expect"], ex["cite"]


def test_apply_D_spec_example_and_matrix():
    g = _gold("spec_grid_examples.json")
    for ex in g["apply_D"]:
        out = grid.apply_D_loop(ex["level"], np.array(ex["v"], float))
        assert np.array_equal(out, np.array(ex["expect"], float)), ex["cite"]
        D = grid.D_matrix(ex["level"])
        assert np.array_equal(D @ np.array(ex["v"], float), np.array(ex["expect"], float))


def test_new_grid_counts():
    g = _gold("spec_grid_examples.json")
    for ex in g["new_grid"]:
        assert grid.side_of(ex["level"]) ** 2 == ex["N"]
        assert list(grid.rowsums(ex["level"]).astype(int)) == ex["neighbor_counts"]


def test_paper_sizes():
    g = _gold("paper_sizes.json")
    assert 12 * grid.side_of(10) ** 2 == g["fullsky_pixels_level10"]["value"]
    assert grid.side_of(10) ** 2 == g["pixels_per_face_level10"]["value"]
    assert 9 * grid.side_of(10) ** 2 == g["nN_planck"]["value"]
    assert 4 * grid.side_of(10) ** 2 == g["mN_planck"]["value"]
    assert [12 * grid.side_of(h) ** 2 for h in (1, 2, 3)] == g["fullsky_pixels_levels_1_2_3"]["value"]


@pytest.mark.parametrize("level", [2, 3, 4])
def test_degree_pattern_and_symmetry(level):
    s = grid.side_of(level)
    deg = grid.rowsums(level).reshape(s, s)
    assert deg[0, 0] == deg[0, -1] == deg[-1, 0] == deg[-1, -1] == 2
    assert np.all(deg[0, 1:-1] == 3) and np.all(deg[1:-1, 0] == 3)
    assert np.all(deg[1:-1, 1:-1] == 4)
    D = grid.D_matrix(level)
    assert (D - D.T).nnz == 0
    assert np.abs(D @ np.ones(s * s)).max() == 0.0          # D 1 = 0
    rng = np.random.default_rng(level)
    v = rng.standard_normal(s * s)
    assert np.allclose(D @ v, grid.apply_D_loop(level, v), rtol=0, atol=1e-13)


@pytest.mark.parametrize("level", [1, 2, 3])
def test_one_zero_eigenvalue(level):
    D = grid.D_matrix(level).toarray()
    ev = np.linalg.eigvalsh(D @ D)
    assert np.sum(np.abs(ev) <= 1e-8 * np.abs(ev).max()) == 1


def test_D2_interior_and_corner_stencil():
    # Closed form: interior row of D^2 has 20 on the diagonal, -8 at the 4 neighbours,
    # 2 at the 4 diagonal pixels and 1 at distance 2 (sum = 0 since D 1 = 0).
    level = 3
    s = grid.side_of(level)
    D = grid.D_matrix(level)
    D2 = (D @ D).toarray()
    j = 3 * s + 3
    row = D2[j].reshape(s, s)
    assert row[3, 3] == 20
    assert row[2, 3] == row[4, 3] == row[3, 2] == row[3, 4] == -8
    assert row[2, 2] == row[2, 4] == row[4, 2] == row[4, 4] == 2
    assert row[1, 3] == row[5, 3] == row[3, 1] == row[3, 5] == 1
    assert abs(row.sum()) == 0
    # corner (0,0): D_00 = -2; (D^2)_00 = 4 + 2 = 6; neighbours -2 + -3 = -5
    c = D2[0].reshape(s, s)
    assert c[0, 0] == 6 and c[0, 1] == -5 and c[1, 0] == -5 and c[1, 1] == 2
    assert c[0, 2] == 1 and c[2, 0] == 1


@pytest.mark.parametrize("level", [2, 3])
def test_laplacian_spectrum_is_textbook_neumann_grid(level):
    # Eigenvalues of the path-graph Laplacian are 2 - 2 cos(pi a / s) (textbook);
    # the grid is the Cartesian product, so its spectrum is the sum.
    L = grid.laplacian(level).toarray()
    ev = np.sort(np.linalg.eigvalsh(L))
    s = grid.side_of(level)
    t = 2 - 2 * np.cos(np.pi * np.arange(s) / s)
    ref = np.sort((t[:, None] + t[None, :]).ravel())
    assert np.allclose(ev, ref, atol=1e-12)
    assert np.allclose(np.sort(exact.face_spectrum(level).ravel()), ref, atol=1e-15)


def test_level_range_errors():
    with pytest.raises(ValueError):
        grid.side_of(13)
    with pytest.raises(IndexError):
        grid.neighbors(1, 4)


def test_nested_index_is_the_z_order_curve():
    """HEALPix NESTED inside a face = Morton / Z-order: level 2 visits the 2x2 blocks in Z order and
    each block in Z order (pixel (x, y) listed by increasing nested index)."""
    order = sorted(((grid.nest_index(2, x, y), (x, y)) for y in range(4) for x in range(4)))
    assert [xy for _, xy in order] == [(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1),
                                       (0, 2), (1, 2), (0, 3), (1, 3), (2, 2), (3, 2), (2, 3), (3, 3)]
    for level in (0, 1, 3, 5):
        idx = grid.pixel_index(level, "nested").reshape(-1)
        assert sorted(idx) == list(range(4 ** level))          # a permutation
    assert grid.nest_index(10, 1023, 1023) == 4 ** 10 - 1


@pytest.mark.parametrize("level", [1, 2, 4])
def test_nested_laplacian_is_the_permuted_row_major_one(level):
    """L_nested = Pi L_row Pi^T with Pi the row-major -> nested permutation (the grid graph does not
    depend on how its vertices are numbered)."""
    perm = grid.pixel_index(level, "nested").reshape(-1)      # perm[row-major j] = nested index
    N = 4 ** level
    Pi = np.zeros((N, N))
    Pi[perm, np.arange(N)] = 1.0
    Ln = grid.laplacian(level, "nested").toarray()
    Lr = grid.laplacian(level).toarray()
    assert np.array_equal(Ln, Pi @ Lr @ Pi.T)
