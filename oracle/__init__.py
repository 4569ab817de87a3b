"""CPU fp64 ORACLE for the Kronecker CG / Sylvester hot path of arxiv 2204.08057.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call or
execute anything in this package.  The product path (``paper_2204_08057_b200``,
``csrc/``) never imports it and shares no code, headers, tables or constants
with it.

Plain, slow, obviously-correct: every operator is the paper's literal sparse
Kronecker matrix assembled with scipy.sparse (PAPER.md Eq.(Q*) P:L73-77,
Eq.(mu*) P:L78-82, Eq.(Axb), B = A (x) I_N P:L53, C = T (x) N P:L111,
Q = P (x) D^2 P:L140-148), and every solver follows the textbook algorithm step
by step in the paper's notation.

Modules
  grid      face grid, neighbour lists, D (Alg.MatvecD)
  model     literal B, C, Q, G = B^T C B + Q, b = B^T C Y; one-by-one row evaluation
  cg        textbook Hestenes-Stiefel CG + single-pass CG variant
  sylvester Sylvester reformulation diagonalised by eigh(M, P) (Lemma 2)
  exact     dense Cholesky (tiny) and DCT-II mode-wise exact solve (hits = 1)

Parity status: every function is pinned by tests/test_oracle_*.py (see DESIGN.md
"Oracle pins"); none is "parity unpinned".
"""

from . import grid, model, cg, sylvester, exact  # noqa: F401
