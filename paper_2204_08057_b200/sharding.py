"""Host-side multi-GPU planning: the 12 independent base faces (App. A) sharded across ranks.

No collective is needed on the data path: faces are independent problems ("repeated 12
times for each base patch"), so each rank batches its faces into one library context and only a
final barrier / max-over-ranks timing crosses ranks.

Load balance: per-face CG iteration counts differ (per-face parameters), and CG iterations grow
like sqrt(cond(G)).  With unit hit counts cond(G) is known in O(k^3) per face from the two
extreme prior eigenvalues (the DCT spectrum of kappa2 + L spans [kappa2, kappa2 + lam_max]):
    cond(G) = lambda_max(M + (kappa2 + lam_max) P) / lambda_min(M + kappa2 P).
Faces are assigned longest-processing-time-first on that cost.
"""

from __future__ import annotations

import math
from typing import List, Sequence

import numpy as np


def face_lam_max(level: int) -> float:
    s = 1 << level
    return 2.0 * (2.0 - 2.0 * math.cos(math.pi * (s - 1) / s)) if s > 1 else 0.0


def patch_cost(level: int, A, noise_prec, prior_scale, kappa2) -> float:
    """sqrt(cond(G)) of one face (unit hits): the CG iteration-count model."""
    A = np.asarray(A, dtype=np.float64)
    M = A.T @ (np.asarray(noise_prec, dtype=np.float64)[:, None] * A)
    P = np.diag(np.asarray(prior_scale, dtype=np.float64))
    lo = np.linalg.eigvalsh(M + kappa2 * P)[0]
    hi = np.linalg.eigvalsh(M + (kappa2 + face_lam_max(level)) * P)[-1]
    return float(math.sqrt(hi / lo))


def assign_lpt(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of units to ``world`` ranks (deterministic)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda j: (load[j], j))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(o) for o in out]


def makespan(costs: Sequence[float], plan: List[List[int]]) -> float:
    return max(sum(costs[i] for i in part) for part in plan) if plan else 0.0


def shard_for_rank(costs: Sequence[float], world: int, rank: int) -> List[int]:
    return assign_lpt(costs, world)[rank]


# ----------------------------------------------------------------------------- slab groups
# With more GPUs than faces can balance (12 faces over 8 GPUs: 1.5 faces each, per-face iteration
# counts 89-319), ranks are grouped: a group of g ranks splits each of its faces into g row slabs
# (kron_cg_create_slab) and faces are assigned to groups by LPT.  A single face
# (planck, stress) is split over all ranks.
# Modelled per-pass cost of the cross-rank exchange (halo rows + scalar sum), in units of one full
# face's CG pass (~40 us on a B200 for N = 4^10, k = 4; the exchange is a few us over NVLink).
SLAB_PASS_OVERHEAD = 0.15


def plan_groups(costs: Sequence[float], world: int):
    """Choose the group size g (a power of two dividing world, <= 8) minimising the modelled
    makespan  max_group(sum cost) / g + SLAB_PASS_OVERHEAD * max_group(max cost) [g > 1]
    (faces of a group iterate together in one batch; converged faces drop out, so the group's
    passes = its slowest face's).  Ties -> smaller g.  Returns (g, faces_per_group) with
    faces_per_group[j] the faces of group j (ranks j*g .. j*g+g-1)."""
    best = None
    g = 1
    while g <= min(world, 8):
        if world % g == 0:
            plan = assign_lpt(costs, world // g)
            t = makespan(costs, plan) / g
            if g > 1:
                t += SLAB_PASS_OVERHEAD * max(max(costs[i] for i in part) for part in plan if part)
            if best is None or t < best[0] - 1e-12:
                best = (t, g, plan)
        g *= 2
    return best[1], best[2]


def rank_role(costs: Sequence[float], world: int, rank: int):
    """(g, group index, slab index within the group, faces of the group) of one rank."""
    g, plan = plan_groups(costs, world)
    return g, rank // g, rank % g, plan[rank // g]
