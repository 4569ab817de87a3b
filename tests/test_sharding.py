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
