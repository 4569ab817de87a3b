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
# Per-pass cost of the cross-rank exchange (halo rows + scalar sum) in units of one full face's CG
# pass (~40 us on a B200 for N = 4^10, k = 4), MEASURED in the one-launch emulation (planck face,
# bench.py "slab_emulation" / scripts/probes/slab_probe.py, profiles/r02/slab_probe_r02.txt):
# +7.9 / +7.4 / +12.5 us per pass for g = 2 / 4 / 8.  Over NVLink add ~1-2 us of link latency.
SLAB_PASS_OVERHEAD = {2: 0.20, 4: 0.19, 8: 0.31}


def _ovh(g: int) -> float:
    return 0.0 if g == 1 else SLAB_PASS_OVERHEAD.get(g, max(SLAB_PASS_OVERHEAD.values()))


def plan_groups(costs: Sequence[float], world: int):
    """Choose the group size g (a power of two dividing world, <= 8) minimising the modelled
    makespan  max_group(sum cost) / g + overhead(g) * max_group(max cost)  (faces of a group iterate
    together in one batch; converged faces drop out, so the group's passes = its slowest face's).
    Ties -> smaller g.  Returns (g, faces_per_group) with faces_per_group[j] the faces of group j
    (ranks j*g .. j*g+g-1)."""
    best = None
    g = 1
    while g <= min(world, 8):
        if world % g == 0:
            plan = assign_lpt(costs, world // g)
            t = uniform_makespan(costs, plan, g)
            if best is None or t < best[0] - 1e-12:
                best = (t, g, plan)
        g *= 2
    return best[1], best[2]


def uniform_makespan(costs: Sequence[float], plan: List[List[int]], g: int) -> float:
    """Modelled time of a uniform plan: groups of g ranks, faces of group j split g ways."""
    return max((sum(costs[i] for i in part) / g + _ovh(g) * max(costs[i] for i in part)) if part else 0.0
               for part in plan)


def mixed_plan(costs: Sequence[float], world: int, g: int = 2):
    """The survey's alternative for more ranks than faces can balance (e.g. 12 faces on 8 GPUs:
    8 whole faces + 4 faces half-split): every rank runs a whole-face context AND its share of a
    g-split context (two launches per step).  The s most expensive faces are split (s chosen by
    the model), the split faces LPT over world/g groups, the whole faces LPT over the ranks on top
    of the split loads.  Returns (modelled makespan, split faces per group, whole faces per rank)."""
    best = None
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    for s in range(0, len(costs) + 1):
        split, whole = order[:s], order[s:]
        groups = assign_lpt([costs[i] for i in split], world // g) if s else [[] for _ in range(world // g)]
        groups = [[split[i] for i in grp] for grp in groups]
        load = []
        for r in range(world):
            part = groups[r // g]
            load.append((sum(costs[i] for i in part) / g + _ovh(g) * max(costs[i] for i in part)) if part else 0.0)
        per_rank = [[] for _ in range(world)]
        for i in whole:  # LPT on top of the split loads
            r = min(range(world), key=lambda j: (load[j], j))
            per_rank[r].append(i)
            load[r] += costs[i]
        t = max(load)
        if best is None or t < best[0] - 1e-12:
            best = (t, groups, [sorted(p) for p in per_rank])
    return best


def rank_role(costs: Sequence[float], world: int, rank: int):
    """(g, group index, slab index within the group, faces of the group) of one rank."""
    g, plan = plan_groups(costs, world)
    return g, rank // g, rank % g, plan[rank // g]
