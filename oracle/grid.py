"""Oracle: one HEALPix base face as a 2^L x 2^L four-neighbour grid, and the matrix D.

PAPER.md:
  * App. A P:L762, P:L772 -- level h has 4^h pixels per base face; each face analysed
    independently (no cross-face neighbours).
  * App. C P:L820 -- neighbours are the 4 pixels sharing an edge.
  * Sec. 3 P:L100-106 -- D_{j1 j2} = 1 for neighbours, 0 otherwise, and the diagonal is
    minus the row sum of the off-diagonals; i.e. D = Adj - Deg = -(graph Laplacian).
  * Alg.MatvecD P:L128-138 -- v(j) <- sum of neighbours - rowsum * v(j).
Readings (R1, R2, R11): row-major pixel order idx = y*side + x (default) or the
HEALPix NESTED order inside a face (the bits of x on the even, of y on the odd positions of idx,
i.e. the Z-order curve; "Find neighbours" works on HEALPix indices); free face boundary
(corner 2, edge 3, interior 4 neighbours); Alg.MatvecD evaluated out-of-place.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def side_of(level: int) -> int:
    if level < 0 or level > 12:
        raise ValueError("level out of range [0, 12]")
    return 1 << level


def nest_index(level: int, x: int, y: int) -> int:
    """HEALPix NESTED index of pixel (x, y) inside a face: bit b of x -> bit 2b, of y -> 2b+1."""
    out = 0
    for b in range(level):
        out |= ((x >> b) & 1) << (2 * b)
        out |= ((y >> b) & 1) << (2 * b + 1)
    return out


def pixel_index(level: int, layout: str = "row"):
    """[side][side] array of the pixel index of (y, x) in the given layout ("row" or "nested")."""
    s = side_of(level)
    if layout == "row":
        return np.arange(s * s).reshape(s, s)
    if layout == "nested":
        return np.array([[nest_index(level, x, y) for x in range(s)] for y in range(s)], dtype=np.int64)
    raise ValueError(f"unknown layout {layout!r}")


def neighbors(level: int, j: int) -> list:
    """In-face edge neighbours of pixel j (row-major), sorted ascending."""
    s = side_of(level)
    if j < 0 or j >= s * s:
        raise IndexError("pixel index out of range")
    y, x = divmod(j, s)
    out = []
    if y > 0:
        out.append(j - s)
    if x > 0:
        out.append(j - 1)
    if x < s - 1:
        out.append(j + 1)
    if y < s - 1:
        out.append(j + s)
    return sorted(out)


def adjacency(level: int, layout: str = "row") -> sp.csr_matrix:
    """Adjacency matrix of the face grid (symmetric 0/1) with pixels numbered in `layout`."""
    s = side_of(level)
    N = s * s
    idx = pixel_index(level, layout)
    rows, cols = [], []
    # horizontal edges (y, x) -- (y, x+1)
    a = idx[:, :-1].ravel()
    b = idx[:, 1:].ravel()
    rows += [a, b]
    cols += [b, a]
    # vertical edges (y, x) -- (y+1, x)
    a = idx[:-1, :].ravel()
    b = idx[1:, :].ravel()
    rows += [a, b]
    cols += [b, a]
    r = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
    c = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    return sp.csr_matrix((np.ones(r.size), (r, c)), shape=(N, N))


def rowsums(level: int, layout: str = "row") -> np.ndarray:
    """Precomputed off-diagonal row sums of D = neighbour counts."""
    return np.asarray(adjacency(level, layout).sum(axis=1)).ravel()


def D_matrix(level: int, layout: str = "row") -> sp.csr_matrix:
    """D with D_ij = 1 for neighbours and D_jj = -sum_{l != j} D_jl."""
    Adj = adjacency(level, layout)
    return (Adj - sp.diags(rowsums(level, layout))).tocsr()


def laplacian(level: int, layout: str = "row") -> sp.csr_matrix:
    """Graph Laplacian L = Deg - Adj = -D."""
    return (-D_matrix(level, layout)).tocsr()


def apply_D_loop(level: int, v: np.ndarray) -> np.ndarray:
    """Alg.MatvecD written out as the pixel loop, out-of-place (reading R11).

    Pure Python; for small faces only.
    """
    s = side_of(level)
    N = s * s
    v = np.asarray(v, dtype=np.float64).reshape(N)
    out = np.empty(N)
    for j in range(N):
        nb = neighbors(level, j)
        out[j] = sum(v[i] for i in nb) - len(nb) * v[j]
    return out
