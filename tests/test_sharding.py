"""Multi-GPU host logic on CPU: face sharding (LPT on the sqrt(cond) cost model), the gloo
world_size-2 version of bench.py's sharded step (no data-path collective; barrier + MAX timing)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2204_08057_b200.sharding import assign_lpt, makespan, patch_cost, shard_for_rank


def test_lpt_covers_each_unit_once_and_is_deterministic():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        costs = list(rng.uniform(1, 10, 12))
        plan = assign_lpt(costs, world)
        assert sorted(i for part in plan for i in part) == list(range(12))
        assert plan == assign_lpt(costs, world)
        assert [shard_for_rank(costs, world, r) for r in range(world)] == plan
        lb = max(sum(costs) / world, max(costs))
        assert makespan(costs, plan) <= 4 / 3 * lb + 1e-12   # Graham's LPT bound
    assert assign_lpt([1.0] * 12, 4) == [[0, 4, 8], [1, 5, 9], [2, 6, 10], [3, 7, 11]]


def test_cost_model_tracks_oracle_iterations():
    from synth import make_patch
    from oracle import cg, model
    costs, its = [], []
    for seed in range(10):
        p = make_patch(5, 9, 4, seed=seed, tau="loguniform")
        costs.append(patch_cost(p.level, p.A, p.noise_prec, p.tau, p.kappa2))
        G, b = model.problem_system(p)
        its.append(cg.cg_hs(G, b, tol=1e-10).iterations)
    rc = np.argsort(np.argsort(costs))
    ri = np.argsort(np.argsort(its))
    spearman = np.corrcoef(rc, ri)[0, 1]
    assert spearman > 0.7, (costs, its)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import time
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth import make_patch
    from oracle import cg, model
    seeds = list(range(20, 26))
    # every rank derives the same plan from the small parameters alone
    params = [make_patch(2, 9, 3, seed=s, tau="loguniform") for s in seeds]
    costs = [patch_cost(3, p.A, p.noise_prec, p.tau, p.kappa2) for p in params]
    mine = shard_for_rank(costs, world, rank)
    dist.barrier()
    t0 = time.perf_counter()
    res = {}
    for i in mine:
        p = make_patch(3, 9, 3, seed=seeds[i], tau="loguniform")
        G, b = model.problem_system(p)
        r = cg.cg_hs(G, b, tol=1e-10)
        res[i] = (r.iterations, r.x)
    dist.barrier()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, res, float(t.item())))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_step_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from synth import make_patch
    from oracle import cg, model
    covered = sorted(i for mine, _, _ in gathered for i in mine)
    assert covered == list(range(6))
    tmax = {t for _, _, t in gathered}
    assert len(tmax) == 1            # every rank holds the same MAX-over-ranks time
    for mine, res, _ in gathered:
        for i in mine:
            p = make_patch(3, 9, 3, seed=20 + i, tau="loguniform")
            G, b = model.problem_system(p)
            r = cg.cg_hs(G, b, tol=1e-10)
            assert res[i][0] == r.iterations
            assert np.array_equal(res[i][1], r.x)


def test_plan_groups_slabs_only_where_faces_cannot_balance():
    from paper_2204_08057_b200.sharding import plan_groups, rank_role
    rng = np.random.default_rng(1)
    costs = list(rng.uniform(9, 18, 12))       # fullsky-like spread (sqrt cond)
    assert plan_groups(costs, 1)[0] == 1
    assert plan_groups(costs, 2)[0] == 1         # 12 faces balance over 2 ranks
    g8, plan8 = plan_groups(costs, 8)
    assert g8 > 1 and len(plan8) == 8 // g8      # 8 ranks: faces must be split to balance
    assert sorted(i for part in plan8 for i in part) == list(range(12))
    assert plan_groups([5.0], 4) == (4, [[0]])   # one face (planck): split over every rank
    roles = [rank_role(costs, 8, r) for r in range(8)]
    assert [r[1] for r in roles] == [r // g8 for r in range(8)] and [r[2] for r in roles] == [r % g8 for r in range(8)]
    assert all(r[3] == plan8[r[1]] for r in roles)


def test_mixed_plan_model():
    """The survey's mixed plan (whole faces + a few split faces per rank) against the uniform group
    plans under the measured per-pass exchange costs (sharding.SLAB_PASS_OVERHEAD)."""
    from paper_2204_08057_b200.sharding import assign_lpt, mixed_plan, plan_groups, uniform_makespan
    rng = np.random.default_rng(1)
    costs = list(rng.uniform(9, 18, 12))
    costs[0] = 30.0                                # one slow face (the fullsky face 0 pattern)
    for world in (2, 4, 8):
        g, plan = plan_groups(costs, world)
        tu = uniform_makespan(costs, plan, g)
        assert tu == min(uniform_makespan(costs, assign_lpt(costs, world // gg), gg)
                         for gg in (1, 2, 4, 8) if world % gg == 0 and gg <= world)
        for gm in (2, 4):
            if world % gm:
                continue
            t, groups, whole = mixed_plan(costs, world, gm)
            faces = sorted([i for grp in groups for i in grp] + [i for w in whole for i in w])
            assert faces == list(range(12))            # every face exactly once
            assert t <= uniform_makespan(costs, assign_lpt(costs, world), 1) + 1e-9  # s = 0 is a candidate
            assert t >= sum(costs) / world - 1e-9      # never below the perfect split
    t8, groups8, _ = mixed_plan(costs, 8, 4)
    assert 0 in groups8[0] + groups8[1]                 # the slow face is the one split


def _slab_worker(rank, world, port, out):
    """Row-slab single-pass CG on CPU (gloo): each rank holds rows [rank R, (rank+1) R) of x, r, p
    plus 2 ghost rows of r and p per side, exchanged every iteration (send/recv), and the three
    CG scalars are summed across ranks (all_reduce) -- the protocol of the slab kernel."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth import make_patch
    from oracle import model
    p = make_patch(4, 9, 3, seed=7, tau="loguniform")
    side, k, Rr, H = p.side, p.k, p.side // world, 2
    M = p.A.T @ np.diag(p.noise_prec) @ p.A
    b = model.assemble_rhs(p.level, p.A, p.noise_prec, p.Y).reshape(k, side, side)
    lo = rank * Rr

    def G(v, g0):  # operator on rows g0.. of a ghosted block (rows outside the face are zero)
        out = np.einsum("cd,dyx->cyx", M, v)
        nb = np.zeros_like(v)
        nb[:, 1:, :] += v[:, :-1, :]; nb[:, :-1, :] += v[:, 1:, :]
        nb[:, :, 1:] += v[:, :, :-1]; nb[:, :, :-1] += v[:, :, 1:]
        gy = np.arange(g0, g0 + v.shape[1])[:, None]
        gx = np.arange(side)[None, :]
        deg = 4 - (gy == 0) - (gy == side - 1) - (gx == 0) - (gx == side - 1)
        return out + p.tau[:, None, None] * ((p.kappa2 + deg)[None] * v - nb)

    def halo(a):  # a: [k][Rr + 2H][side]; fill ghost rows from the neighbours
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(a[:, H:2 * H].copy()), rank - 1),
                    dist.P2POp(dist.irecv, up := torch.empty(k, H, side, dtype=torch.float64), rank - 1)]
        if rank < world - 1:
            ops += [dist.P2POp(dist.isend, torch.from_numpy(a[:, Rr:Rr + H].copy()), rank + 1),
                    dist.P2POp(dist.irecv, dn := torch.empty(k, H, side, dtype=torch.float64), rank + 1)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if rank > 0:
            a[:, :H] = up.numpy()
        if rank < world - 1:
            a[:, Rr + H:] = dn.numpy()

    def allsum(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.tolist()

    inside = (np.arange(lo - H, lo + Rr + H) >= 0) & (np.arange(lo - H, lo + Rr + H) < side)
    r = np.zeros((k, Rr + 2 * H, side)); r[:, H:H + Rr] = b[:, lo:lo + Rr]
    pp = np.zeros_like(r)
    x = np.zeros((k, Rr, side))
    halo(r)
    alpha = beta = 0.0
    gamma = bn2 = None
    its = 0
    for it in range(-1, 400):
        pn = r + beta * pp
        pn[:, ~inside] = 0.0
        q = G(pn, lo - H)
        rn = r - alpha * q
        rn[:, ~inside] = 0.0
        w = G(rn, lo - H)
        own = slice(H, H + Rr)
        rr, wr = allsum([float((rn[:, own] ** 2).sum()), float((w[:, own] * rn[:, own]).sum())])
        x += alpha * pn[:, own]
        r, pp = rn, pn
        r[:, :H] = r[:, Rr + H:] = 0.0
        pp[:, :H] = pp[:, Rr + H:] = 0.0
        halo(r); halo(pp)
        if it < 0:
            bn2, gamma, alpha = rr, rr, rr / wr
            continue
        its = it + 1
        if rr <= 1e-20 * bn2:
            break
        beta = rr / gamma
        alpha, gamma = rr / (wr - beta * rr / alpha), rr
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, its, x))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_row_slab_cg_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from synth import make_patch
    from oracle import cg, model
    p = make_patch(4, 9, 3, seed=7, tau="loguniform")
    G, b = model.problem_system(p)
    ref = cg.cg_single_pass(G, b, tol=1e-10)
    gathered.sort()
    x = np.concatenate([g[2] for g in gathered], axis=1).reshape(-1)
    assert gathered[0][1] == gathered[1][1]
    assert abs(gathered[0][1] - ref.iterations) <= 1
    assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-9


def test_exchange_records_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_records_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = [bytes([r]) * 64 + (4096 * r + 256).to_bytes(8, "little") for r in range(world)]
    for rank, recs in res:
        assert recs == expect


def _records_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import importlib.util, sys
    # the record exchange is plain torch.distributed host logic; load the binding module's helper
    # without loading the CUDA library (no GPU here)
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2204_08057_b200", "kroncg.py")).read()
    start = src.index("def exchange_records(")
    end = src.index("\n\n\n", start)
    ns = {}
    exec(src[start:end], ns)
    rec = bytes([rank]) * 64 + (4096 * rank + 256).to_bytes(8, "little")
    out.put((rank, ns["exchange_records"](rec)))
    dist.barrier()
    dist.destroy_process_group()
