#!/usr/bin/env python
"""Benchmark of the hot path: full-sky (12 faces, L=10, n=9, k=4) posterior-mean solves on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]
                    [--config fullsky|planck|medium|tiny|stress] [--route kron|sylvester]

One "step" = one full pass of the hot path over one batch of synthetic input: the right-hand side
(a2), the whole CG iteration (a3-a5) to tolerance 1e-10 for every face, the termination report with
the true residual (a7), all faces batched in one launch per rank (a8).  The Sylvester route (a6) is
timed in the same run and reported under "sylvester"; the paper's block-Lanczos Sylvester solver
(Alg. SylvSolver) under "lanczos" (its own context: HBM-resident basis).  Faces are sharded across ranks (LPT on the
sqrt(cond) cost model); there is no data-path collective, only the timing barrier/max.

`value` is whole-job full-sky solves/s (device time, CUDA events on the launching stream, max over
ranks).  Inputs (Y: 0.9 GB, solver state: 1.6 GB) are larger than the 126 MB L2, so no flush is
needed between steps.  --impl reference times the CPU fp64 oracle (scipy, literal Kronecker
assembly) on a bounded sample of the same workload and extrapolates to full-sky solves/s.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "CG iters/s and full-sky solves/s at 1/2/4/8 B200; achieved HBM GB/s vs peak"
TOL = 1e-10


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(workload: str, route: str):
    """dram bytes per launch of the CG kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(f"{workload}/{route}")
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(dev_index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _patches_for(config: str, world: int, rank: int):
    """This rank's faces and role.  Faces are grouped (sharding.plan_groups): a group of g ranks
    batches its faces in one context and, for g > 1, splits every face into g row slabs (one per
    rank of the group).  Returns (problems of the group, their indices, costs, g, slab index)."""
    from synth import CONFIGS
    from synth.problems import make_patch
    from paper_2204_08057_b200.sharding import patch_cost, rank_role
    c = CONFIGS[config]
    if world == 1:
        probs = [make_patch(c["level"], c["n"], c["k"], sd, tau=c["tau"], kappa2=c["kappa2"]) for sd in c["seeds"]]
        costs = [patch_cost(c["level"], p.A, p.noise_prec, p.tau, p.kappa2) for p in probs]
        return probs, list(range(len(probs))), costs, 1, 0
    # the cost model needs only the small parameters (identical draws at a tiny level); full
    # problems are drawn for this rank's group only
    probs_all = [make_patch(min(c["level"], 2), c["n"], c["k"], sd, tau=c["tau"], kappa2=c["kappa2"])
                 for sd in c["seeds"]]
    costs = [patch_cost(c["level"], p.A, p.noise_prec, p.tau, p.kappa2) for p in probs_all]
    g, grp, slab, mine = rank_role(costs, world, rank)
    probs = [make_patch(c["level"], c["n"], c["k"], c["seeds"][i], tau=c["tau"], kappa2=c["kappa2"]) for i in mine]
    return probs, mine, costs, g, slab


def _slab_probe(dev, G=8, steps=5):
    """Cost of the row-slab machinery on one GPU: the planck face (L=10, k=4) solved unsplit and
    split into G row slabs with all G ranks emulated in one cooperative launch (halo rows through
    the neighbours' ghost rows, per-iteration cross-rank scalar sums through slots + flags).  On a
    real G-GPU run each rank does 1/G of the bytes; here one GPU does all of them, so the per-pass
    difference is the protocol's overhead."""
    import torch
    from synth import make_config
    from synth.problems import stack
    from paper_2204_08057_b200.kroncg import KronCG, KronCGSlab, split_rows
    p = make_config("planck")[0]
    st = stack([p])
    Y = torch.from_numpy(st["Y"]).to(dev)
    c1 = KronCG(p.level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev)
    cs = KronCGSlab(p.level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], G, emulate=True, device=dev)
    Ys = split_rows(Y, G)
    out = {"config": "planck", "slabs": G}
    for name, fn in (("unsplit", lambda: c1.solve(Y, tol=TOL)[1]), ("slab", lambda: cs.solve(Ys, tol=TOL)[1])):
        for _ in range(2):
            fn()
        reps = [fn() for _ in range(steps)]
        lt = sum(r["loop_time_s"] for r in reps) / steps
        it = reps[-1]["iterations"]
        out[name] = {"solves_per_s": steps / sum(r["wall_time_s"] for r in reps), "iterations": it,
                     "cg_kernel_us_per_pass": lt / (it + 1) * 1e6}
    out["overhead_us_per_pass"] = out["slab"]["cg_kernel_us_per_pass"] - out["unsplit"]["cg_kernel_us_per_pass"]
    return out


def _oracle_iterations(config):
    p = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(config, {}).get("kron_cg_iterations")


def _cpu_baseline(problems, gpu_iters_per_patch, budget_s=20.0):
    """Oracle (as it stands) on a bounded sample: assemble face 0 literally, run textbook CG for a
    bounded number of iterations, extrapolate to one full-sky solve with the measured per-face
    iteration counts.  BLAS limited to 1 thread (scipy SpMV is single-threaded)."""
    from threadpoolctl import threadpool_limits
    from oracle import cg, model
    p = problems[0]
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        G, b = model.problem_system(p)
        t_asm = time.perf_counter() - t0
        n_it = 0
        t1 = time.perf_counter()
        # time single iterations until the budget is used
        probe = cg.cg_hs(G, b, tol=TOL, max_iter=2)
        t_two = time.perf_counter() - t1
        per = max(t_two / 2, 1e-6)
        n_it = int(max(2, min(400, (budget_s - t_asm) / per)))
        t2 = time.perf_counter()
        res = cg.cg_hs(G, b, tol=TOL, max_iter=n_it)
        t_it = (time.perf_counter() - t2) / max(res.iterations, 1)
        del probe
    n_faces = len(gpu_iters_per_patch)
    total_its = sum(gpu_iters_per_patch)   # GPU counts (equal to the oracle's, see parity tests)
    t_sky = n_faces * t_asm + total_its * t_it
    return {"value": 1.0 / t_sky, "unit": "full-sky solves/s", "cores": 1, "kind": "oracle",
            "sample": (f"oracle (scipy CSR, literal Kronecker assembly, textbook HS-CG) on face 0 of "
                       f"{len(problems)}: assembly {t_asm:.2f} s + {res.iterations} CG iterations "
                       f"({t_it * 1e3:.1f} ms/iter, L={p.level}, k={p.k}); extrapolated to "
                       f"{n_faces} faces x assembly + {total_its} face-iterations"),
            "s_per_face_iteration": t_it, "s_assembly": t_asm,
            "cg_iters_per_s": 1.0 / t_it}


def _cpu_baseline_lanczos(problems, steps_per_face, budget_steps=None):
    """Oracle block Lanczos (oracle.lanczos, Alg. SylvSolver step by step, numpy/scipy as it stands)
    on face 0 to convergence, 1 BLAS thread; extrapolated to the full sky by the faces' step counts
    (its per-step cost grows with the step: eigh of T_i every step, so this is an estimate)."""
    from threadpoolctl import threadpool_limits
    from oracle import lanczos
    p = problems[0]
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        r = lanczos.problem_solve(p, tol=TOL, max_iter=budget_steps or 100000)
        t = time.perf_counter() - t0
    per_step = t / max(r.iterations, 1)
    t_sky = per_step * sum(steps_per_face)
    return {"value": 1.0 / t_sky, "unit": "full-sky solves/s", "cores": 1, "kind": "oracle",
            "sample": (f"oracle.lanczos (Alg. SylvSolver, literal sparse N^-1 Q0, eigh of T_i per step) on face 0 "
                       f"of {len(problems)}: {r.iterations} steps in {t:.2f} s (L={p.level}, k={p.k}); "
                       f"extrapolated to {sum(steps_per_face)} face-steps"),
            "s_face0": t}


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from synth import CONFIGS
    from synth.problems import make_patch
    from threadpoolctl import threadpool_limits
    from oracle import cg, model
    c = CONFIGS[args.config]
    p = make_patch(c["level"], c["n"], c["k"], c["seeds"][0], tau=c["tau"], kappa2=c["kappa2"])
    n_faces = len(c["seeds"])
    iters_sample = args.ref_iters
    times = []
    with threadpool_limits(limits=1):
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            G, b = model.problem_system(p)
            t_asm = time.perf_counter() - t0
            t1 = time.perf_counter()
            res = cg.cg_hs(G, b, tol=TOL, max_iter=iters_sample)
            t_it = (time.perf_counter() - t1) / max(res.iterations, 1)
            if step >= args.warmup:
                times.append((t_asm, t_it))
    t_asm = statistics.mean(t for t, _ in times)
    t_it = statistics.mean(t for _, t in times)
    # extrapolation to one full solve with the ORACLE's own per-face iteration counts
    # (tests/golden/oracle_iterations.json, written by scripts/oracle_iterations.py from oracle/)
    its_faces = _oracle_iterations(args.config) or [args.ref_face_iters] * n_faces
    t_sky = n_faces * t_asm + sum(its_faces) * t_it
    val = 1.0 / t_sky
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "full-sky solves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_sky * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/ recipe, SURVEY 8(d)); CPU fp64 oracle",
        "config": {"workload": args.config, "level": c["level"], "n": c["n"], "k": c["k"],
                   "patches": n_faces, "tol": TOL, "route": "kron"},
        "cpu_baseline": {"value": val, "unit": "full-sky solves/s", "cores": 1, "kind": "oracle",
                         "sample": (f"per step: literal assembly of face 0 + {iters_sample} textbook "
                                    f"CG iterations (1 thread); extrapolated as {n_faces} faces x "
                                    f"assembly + {sum(its_faces)} oracle face-iterations")},
        "e2e": {"value": val, "unit": "full-sky solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "cg_iters_per_s": 1.0 / t_it,
    }
    print(json.dumps(line), flush=True)
    return 0


def _lanczos_leg(problems, st, dev, timed, args, cpu=False):
    """The paper's block-Lanczos Sylvester solver (Alg. SylvSolver, sylvester_lanczos_solve) on this
    rank's faces: HBM-resident basis (lanczos_store) sized for the oracle's step counts, inputs
    resident; its own context (the basis is not part of the CG workspace)."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev,
                 lanczos_cap=args.lanczos_cap, lanczos_store=True)
    Y = torch.from_numpy(st["Y"]).to(dev)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    fn = lambda: ctx.lanczos(Y, mu, tol=TOL)[1]
    for _ in range(max(1, args.warmup)):
        r = fn()
        assert r["converged"], r
    t, reps = timed(fn, args.steps)
    peak, peak_src = _peaks()
    b = sum(r["loop_bytes"] for r in reps)
    tl = sum(r["loop_time_s"] for r in reps)
    out = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
           "unit": "full-sky solves/s" if args.config == "fullsky" else "solves/s",
           "lanczos_steps_per_face": reps[-1]["iterations_per"], "mode": "hbm-resident basis (lanczos_store)",
           "true_rel_residual": reps[-1]["rel_residual_true"],
           "roofline": {"bound": "hbm", "achieved": b / tl / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": b / tl / 1e9 / peak, "traffic": _traffic(args.config, "lanczos"),
                        "traffic_note": "ncu dram bytes of the lanczos_kernel launch alone (profiles/ncu_traffic.json)",
                        "kernel": "lanczos_kernel + lz_assemble_kernel", "peak_source": peak_src,
                        "algorithmic_bytes_per_launch": b / len(reps), "avg_launch_ms": tl / len(reps) * 1e3}}
    if cpu and not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_baseline_lanczos(problems, reps[-1]["iterations_per"])
    del ctx
    torch.cuda.empty_cache()
    # the paper's memory-lean mode: four block slots, M assembled by a second Lanczos pass
    ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev,
                 lanczos_cap=args.lanczos_cap, lanczos_store=False)
    fn = lambda: ctx.lanczos(Y, mu, tol=TOL)[1]
    fn()
    t2, reps2 = timed(fn, args.steps)
    b2 = sum(r["loop_bytes"] for r in reps2)
    tl2 = sum(r["loop_time_s"] for r in reps2)
    out["replay_mode"] = {"value": len(reps2) / t2, "ms_per_step": t2 / len(reps2) * 1e3,
                          "mode": "second Lanczos pass (P:L520-528), 4 block slots",
                          "roofline_frac": b2 / tl2 / 1e9 / peak}
    del ctx, Y, mu
    torch.cuda.empty_cache()
    return out


def _pcg_leg(problems, st, dev, timed, args):
    """Pixel-block-Jacobi preconditioned CG (reading R10; the paper: preconditioners "can be used",
    P:L245) on this rank's faces: same metric, fewer iterations, same kernel structure."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev,
                 precond="block_jacobi")
    Y = torch.from_numpy(st["Y"]).to(dev)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    fn = lambda: ctx.solve(Y, mu, tol=TOL)[1]
    r = fn()
    assert r["converged"], r["status_name"]
    t, reps = timed(fn, args.steps)
    peak, peak_src = _peaks()
    b = sum(r["loop_bytes"] for r in reps)
    tl = sum(r["loop_time_s"] for r in reps)
    out = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
           "unit": "full-sky solves/s" if args.config == "fullsky" else "solves/s",
           "face_iterations_per_solve": reps[-1]["system_iterations"], "iterations_per_face": reps[-1]["iterations_per"],
           "true_rel_residual": reps[-1]["rel_residual_true"],
           "roofline": {"bound": "hbm", "achieved": b / tl / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": b / tl / 1e9 / peak, "traffic": None, "kernel": "cg_persistent_kernel (PREC)",
                        "peak_source": peak_src}}
    del ctx, Y, mu
    torch.cuda.empty_cache()
    return out


def _variance_leg(ctx, timed, args, n_probes=4):
    """Posterior variances (posterior_variance: Hutchinson) on this rank's faces:
    one step = n_probes probes, each one batched CG solve of every face with b = the probe."""
    fn = lambda: ctx.posterior_variance(n_probes, seed=11, tol=TOL)[1]
    r = fn()
    assert r["status"] == 0, r["status_name"]
    t, reps = timed(fn, max(1, args.steps // 2))
    peak, peak_src = _peaks()
    b = sum(r["loop_bytes"] for r in reps)
    tl = sum(r["loop_time_s"] for r in reps)
    return {"value": len(reps) * n_probes / t, "unit": "probe solves/s (all faces of the rank per probe)",
            "probes_per_step": n_probes, "ms_per_step": t / len(reps) * 1e3,
            "face_iterations_per_probe": reps[-1]["system_iterations"] / n_probes,
            "roofline": {"bound": "hbm", "achieved": b / tl / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": b / tl / 1e9 / peak, "traffic": None, "kernel": "cg_persistent_kernel",
                         "peak_source": peak_src}}


def _paper_leg(dev, timed, args, level=10, faces=12):
    """The paper's own workload on the full sky: App. B physical A and printed T,
    phi = 1, Q0 = D^2 with kappa2 = 0, random hits 1..4, HEALPix NESTED order, 12 faces at level 10
    (seeds 400..411), through all three routes (inputs resident)."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.physics import make_paper_patch, nested_order
    from synth.problems import stack
    ps = [make_paper_patch(level, seed=400 + f) for f in range(faces)]
    st = stack(ps)
    hits = torch.from_numpy(nested_order(st["hits"])).to(dev)
    Y = torch.from_numpy(nested_order(st["Y"])).to(dev)
    ctx = KronCG(level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=hits, device=dev,
                 layout="nested", prior="d2", lanczos_cap=64, lanczos_store=True)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    out = {"workload": f"paper: App. B A and T, phi = 1, D^2 prior kappa2 = 0, hits 1..4, NESTED; "
                       f"{faces} faces, level {level}", "unit": "full-sky solves/s"}
    for name, fn in (("kron", ctx.solve), ("sylvester", ctx.sylvester), ("lanczos", ctx.lanczos)):
        call = lambda: fn(Y, mu, tol=TOL)[1]
        r = call()
        assert r["converged"], (name, r["status_name"])
        t, reps = timed(call, args.steps)
        out[name] = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
                     "iterations_per_system": reps[-1]["iterations_per"],
                     "true_rel_residual": reps[-1]["rel_residual_true"]}
    del ctx, Y, mu, hits
    torch.cuda.empty_cache()
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    world, rank, local = _dist()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2204_08057_b200 import build
    if rank == 0 or world == 1:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.problems import stack

    problems, mine, costs, g, slab = _patches_for(args.config, world, rank)
    st = stack(problems)
    if g == 1:
        ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                     device=dev, host_staging=True)
        Yn = st["Y"]
    else:
        # every rank creates every group (same order), then joins its own: slabs of its group's faces
        from paper_2204_08057_b200.kroncg import KronCGSlab, split_rows
        groups = [dist.new_group(list(range(j * g, (j + 1) * g))) for j in range(world // g)]
        ctx = KronCGSlab(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], g,
                         emulate=False, group=groups[rank // g], device=dev, host_staging=True)
        Yn = split_rows(st["Y"], g)[slab:slab + 1]
    Y = torch.from_numpy(Yn).to(dev)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    Y_host = torch.from_numpy(Yn).pin_memory()
    mu_host = torch.empty(mu.shape, dtype=torch.float64).pin_memory()
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps):
        reps = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            reps.append(fn())
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t = e0.elapsed_time(e1) / 1e3
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t, reps

    kron = lambda: ctx.solve(Y, mu, tol=TOL)[1]
    syl = lambda: ctx.sylvester(Y, mu, tol=TOL)[1]
    host = lambda: ctx.solve_host(Y_host, mu_host, tol=TOL)[1]
    main_fn = kron if args.route == "kron" else syl
    other_fn = syl if args.route == "kron" else kron

    for _ in range(args.warmup):
        r = main_fn()
        assert r["converged"], r
    clk = ClockSampler(local)
    t_main, reps = timed(main_fn, args.steps)
    clocks = clk.stop()
    for _ in range(max(1, args.warmup // 2)):
        other_fn()
    t_other, reps_other = timed(other_fn, args.steps)
    host()
    t_e2e, reps_e2e = timed(host, max(1, args.e2e_steps))
    lz = None
    if g == 1 and not args.no_lanczos:
        lz = _lanczos_leg(problems, st, dev, timed, args, cpu=(world == 1))
    pcg = None
    if g == 1 and not args.no_pcg:
        pcg = _pcg_leg(problems, st, dev, timed, args)
    koh = None
    if g == 1 and not args.no_kohler:  # Alg. Kohler (NEXT-4): k sequential batched column solves
        call = lambda: ctx.kohler(Y, mu, tol=TOL)[1]
        rk = call()
        assert rk["converged"], rk["status_name"]
        tk, reps_k = timed(call, args.steps)
        pk, pk_src = _peaks()
        bk = sum(r["loop_bytes"] for r in reps_k)
        tlk = sum(r["loop_time_s"] for r in reps_k)
        koh = {"value": len(reps_k) / tk, "ms_per_step": tk / len(reps_k) * 1e3,
               "system_iterations_per_solve": reps_k[-1]["system_iterations"],
               "roofline": {"bound": "hbm", "achieved": bk / tlk / 1e9, "peak": pk, "unit": "GB/s",
                            "frac": bk / tlk / 1e9 / pk, "traffic": None,
                            "kernel": "cg_persistent_kernel (K = 1, one launch per column) + column kernels",
                            "peak_source": pk_src}}
    var = None
    if g == 1 and not args.no_variance:
        var = _variance_leg(ctx, timed, args)
    paper = None
    if world == 1 and not args.no_paper:
        paper = _paper_leg(dev, timed, args)

    def agg(reps_, t):
        # whole-job numbers: gather per-rank sums
        loc = torch.tensor([sum(r["loop_bytes"] for r in reps_), sum(r["loop_time_s"] for r in reps_),
                            sum(r["system_iterations"] for r in reps_), len(reps_),
                            sum(r["system_iterations"] + r["n_systems"] for r in reps_),
                            1.0 if slab == 0 else 0.0],
                           dtype=torch.float64, device=dev)
        if world > 1:
            allv = [torch.zeros_like(loc) for _ in range(world)]
            dist.all_gather(allv, loc)
        else:
            allv = [loc]
        return [v.tolist() for v in allv]

    g_main = agg(reps, t_main)
    g_other = agg(reps_other, t_other)
    io = torch.tensor([float(Y_host.numel() * 8), float(mu_host.numel() * 8)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(io)  # whole-job bytes moved by the e2e step (every rank's own slab / faces)
    h2d_bytes, d2h_bytes = int(io[0].item()), int(io[1].item())
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_src = _peaks()
    K = args.steps

    gsz = g

    def roofline(g, route):
        # dominant kernel = cg_persistent_kernel; rank 0's launches (CUDA events around it).
        # achieved = the bytes this implementation's pass structure must move (report.loop_bytes:
        # r, p read + written every pass, x read + written every other pass = 40 K N B per
        # iteration on average) / kernel time.  model_48kN = SURVEY 8(d)'s B_min = 48 K N B per
        # pass (x every pass) over the same time: the iteration rate as a fraction of that roofline.
        bytes_, tsec = g[0][0], g[0][1]
        ach = bytes_ / tsec / 1e9 if tsec > 0 else 0.0
        kk = problems[0].k if route == "kron" else 1
        b48 = 48.0 * kk * problems[0].side ** 2 / gsz * g[0][4]
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _traffic(args.config, route), "kernel": "cg_persistent_kernel",
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_ / max(g[0][3], 1),
                "avg_launch_ms": tsec / max(g[0][3], 1) * 1e3,
                "model_48kN": {"bytes_per_launch": b48 / max(g[0][3], 1),
                               "frac": (b48 / tsec / 1e9) / peak if tsec > 0 else 0.0}}

    sys_its_main = sum(v[2] for v in g_main if v[5] > 0) / K  # each group's faces counted once
    line = {
        "metric": METRIC,
        "value": K / t_main,
        "unit": "full-sky solves/s" if args.config == "fullsky" else "solves/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": t_main / K * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/ recipe of SURVEY 8(d), seeds per BASELINE config)",
        "config": {"workload": args.config, "level": problems[0].level, "n": problems[0].n,
                   "k": problems[0].k, "patches": len(costs), "tol": TOL, "route": args.route,
                   "parallelism": f"face-shard{world}" if g == 1 else f"face-groups{world // g}x-rowslab{g}",
                   "l2": "no flush: inputs (Y) and solver state exceed the 126 MB L2"},
        "cg_iters_per_s": sys_its_main * K / t_main,
        "face_iterations_per_solve": sys_its_main,
        "iterations_per_face_rank0": reps[-1]["iterations_per"],
        "roofline": roofline(g_main, args.route),
        "e2e": {"value": len(reps_e2e) / t_e2e, "unit": "full-sky solves/s",
                "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes,
                "api": "kron_cg_solve_host (C ABI, pinned host buffers)"},
        # per solve: rhs, CG, x fix-up, residual apply + reduce (+ back-transform, Sylvester)
        "gpu_launches": K * (6 if args.route == "sylvester" else 5),
        "clocks": clocks,
        "sylvester" if args.route == "kron" else "kron": {
            "value": K / t_other, "ms_per_step": t_other / K * 1e3,
            "system_iterations_per_solve": sum(v[2] for v in g_other if v[5] > 0) / K,
            "roofline": roofline(g_other, "sylvester" if args.route == "kron" else "kron")},
        "true_rel_residual": reps[-1]["rel_residual_true"],
    }
    if lz is not None:
        line["lanczos"] = lz
    if paper is not None:
        line["paper_workload"] = paper
    if var is not None:
        line["posterior_variance"] = var
    if pcg is not None:
        line["pcg_block_jacobi"] = pcg
    if koh is not None:
        line["kohler"] = koh
    if world == 1 and not args.no_slab_probe:
        line["slab_emulation"] = _slab_probe(dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(problems, reps[-1]["iterations_per"])
        if var is not None:  # the oracle's Hutchinson probe = one oracle CG solve per face
            cb = line["cpu_baseline"]
            t_probe = len(problems) * cb["s_assembly"] + var["face_iterations_per_probe"] * cb["s_per_face_iteration"]
            var["cpu_baseline"] = {"value": 1.0 / t_probe, "unit": var["unit"], "cores": 1, "kind": "oracle",
                                   "sample": "oracle.variance.hutchinson = oracle.cg.cg_hs per probe and face; "
                                             "timed by the Kron-CG sample above (same CG, same operator)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="fullsky", choices=["tiny", "medium", "planck", "fullsky", "stress"])
    ap.add_argument("--route", default="kron", choices=["kron", "sylvester"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-slab-probe", action="store_true")
    ap.add_argument("--no-lanczos", action="store_true", help="skip the block-Lanczos (Alg. SylvSolver) leg")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper-workload leg (App. B physics, D^2)")
    ap.add_argument("--no-variance", action="store_true", help="skip the posterior-variance (Hutchinson) leg")
    ap.add_argument("--no-pcg", action="store_true", help="skip the block-Jacobi preconditioned CG leg")
    ap.add_argument("--no-kohler", action="store_true", help="skip the Alg. Kohler leg")
    ap.add_argument("--lanczos-cap", type=int, default=128,
                    help="Lanczos steps provisioned (HBM-resident basis: P k N 8 (cap + 1) bytes)")
    ap.add_argument("--ref-iters", type=int, default=8, help="oracle CG iterations per reference step")
    ap.add_argument("--ref-face-iters", type=int, default=180,
                    help="fallback iterations per face if tests/golden/oracle_iterations.json lacks the config")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
