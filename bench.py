#!/usr/bin/env python
"""Benchmark of the hot path: full-sky (12 faces, L=10, n=9, k=4) posterior-mean solves on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]
                    [--config fullsky|planck|medium|tiny|stress] [--route kron|sylvester]

One "step" = one full pass of the hot path over one batch of synthetic input: the right-hand side
(a2), the whole CG iteration (a3-a5) to tolerance 1e-10 for every face, the termination report with
the true residual (a7), all faces batched in one launch per rank (a8).  Further legs of the same
run, each with its own value, roofline and (where timed) clocks: the Sylvester route (a6,
"sylvester"), the paper's block-Lanczos Sylvester solver (Alg. SylvSolver, "lanczos"), the textbook
HS CG variant ("hs_variant", reading R9), block-Jacobi PCG, Alg. Kohler, posterior variances, the
paper's own workload, the planck face alone ("planck": the north star's >= 70 % config) and the
small-problem regime ("small": tiny and medium, CG state resident in shared memory).  Faces are
sharded across ranks (LPT on the sqrt(cond) cost model); there is no data-path collective, only the
timing barrier/max.

`value` is whole-job full-sky solves/s (device time, CUDA events on the launching stream, max over
ranks).  Inputs (Y: 0.9 GB, solver state: 1.6 GB) are larger than the 126 MB L2, so no flush is
needed between steps.  `e2e` is the same metric through the pipelined host entry point
(kron_cg_solve_host_many: pinned host Y in, mu out, every step's copies inside the timed region,
overlapped with the neighbouring steps' solves).

--impl reference times the CPU fp64 oracle (scipy, literal Kronecker assembly, textbook CG) on a
bounded sample of the same workload -- a pool of min(12, cores) processes, each assembling its faces
and timing a few CG iterations -- extrapolated to one full-sky solve with the ORACLE's own per-face
iteration counts (tests/golden/oracle_iterations.json).

Every roofline is printed three ways: `frac` = the SURVEY 8(d) model (B_min = 48 K N bytes per
system-pass: x, r, p read and written once) over the measured kernel time; `bytes_moved` = the bytes
the implementation's pass structure moves (report.loop_bytes: x every other pass, 40 K N); `ncu_dram`
= the ncu-measured DRAM bytes of the same launch (profiles/ncu_traffic.json) over the same time.
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


def _traffic(key: str):
    """ncu DRAM bytes per launch of a leg's dominant kernel (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(key)
    return v.get("dram_bytes_per_launch") if isinstance(v, dict) else None


def roof3(reps, K, N, kernel, traffic_key=None, model_bytes=None, bound="hbm", note=None):
    """Roofline of a leg's dominant kernel, three ways (module docstring).  reps: solve reports of the
    timed steps (one kernel launch each); K planes per system; N pixels per plane; model_bytes: the
    SURVEY 8(d) algorithmic bytes of the timed launches (default 48 K N per system-pass)."""
    peak, src = _peaks()
    n = max(len(reps), 1)
    t = sum(r["loop_time_s"] for r in reps)
    passes = sum(r["system_iterations"] + r["n_systems"] for r in reps)
    b48 = model_bytes if model_bytes is not None else 48.0 * K * N * passes
    moved = sum(r["loop_bytes"] for r in reps)
    ach = b48 / t / 1e9 if t > 0 else 0.0
    out = {"bound": bound, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
           "traffic": None, "kernel": kernel, "peak_source": src,
           "model": "SURVEY 8(d) B_min = 48 K N bytes per system-pass" if model_bytes is None else "leg's algorithmic bytes",
           "algorithmic_bytes_per_launch": b48 / n, "avg_launch_ms": t / n * 1e3,
           "bytes_moved": {"per_launch": moved / n, "achieved": moved / t / 1e9 if t > 0 else 0.0,
                           "frac": moved / t / 1e9 / peak if t > 0 else 0.0}}
    tr = _traffic(traffic_key) if traffic_key else None
    if tr:
        out["traffic"] = tr
        out["ncu_dram"] = {"per_launch": tr, "achieved": tr / (t / n) / 1e9, "frac": tr / (t / n) / 1e9 / peak,
                           "source": f"profiles/ncu_traffic.json[{traffic_key}]"}
    if note:
        out["note"] = note
    return out


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
            time.sleep(0.3)  # the first sample lands before the timed region starts
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
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _patches_for(config: str, world: int, rank: int, shard_only: bool = False):
    """This rank's faces and role.  Faces are grouped (sharding.plan_groups): a group of g ranks
    batches its faces in one context and, for g > 1, splits every face into g row slabs (one per
    rank of the group).  shard_only: whole faces only (g = 1).  Returns (problems of the group,
    their indices, costs, g, slab index)."""
    from synth import CONFIGS
    from synth.problems import make_patch
    from paper_2204_08057_b200.sharding import assign_lpt, patch_cost, rank_role
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
    if shard_only:
        g, slab, mine = 1, 0, assign_lpt(costs, world)[rank]
    else:
        g, grp, slab, mine = rank_role(costs, world, rank)
    probs = [make_patch(c["level"], c["n"], c["k"], c["seeds"][i], tau=c["tau"], kappa2=c["kappa2"]) for i in mine]
    return probs, mine, costs, g, slab


# ------------------------------------------------------------------------------ CPU oracle pool
def _oracle_worker(conn, config, faces):
    """One oracle process: assemble its faces literally (timed), then time `n` textbook CG iterations
    per face on request.  BLAS limited to one thread (the scipy SpMV is single-threaded)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
        from synth import make_config
        from oracle import cg, model
        systems, asm = {}, {}
        for i in faces:
            p = make_config(config, patches=[i])[0]
            t0 = time.perf_counter()
            systems[i] = model.problem_system(p)
            asm[i] = time.perf_counter() - t0
        conn.send(asm)
        while True:
            n = conn.recv()
            if n is None:
                break
            out = {}
            for i in faces:
                G, b = systems[i]
                t0 = time.perf_counter()
                r = cg.cg_hs(G, b, tol=TOL, max_iter=n)
                out[i] = (time.perf_counter() - t0) / max(r.iterations, 1)
            conn.send(out)


def _oracle_iterations(config):
    p = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get(config, {}).get("kron_cg_iterations")


class OraclePool:
    """min(12, cores) oracle processes over the config's faces (LPT on the oracle's own iteration
    counts); extrapolates a bounded sample to one solve of every face: per worker the sum over its
    faces of (assembly + oracle iterations x time per iteration), the slowest worker = the solve."""

    def __init__(self, config):
        import multiprocessing as mp
        from synth import CONFIGS
        from paper_2204_08057_b200.sharding import assign_lpt
        n_faces = len(CONFIGS[config]["seeds"])
        self.config = config
        self.its = _oracle_iterations(config) or [180] * n_faces
        self.workers = max(1, min(12, len(os.sched_getaffinity(0)), n_faces))
        self.plan = [p for p in assign_lpt([float(v) for v in self.its], self.workers) if p]
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        for faces in self.plan:
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_oracle_worker, args=(b, config, faces), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        self.asm = {}
        for c in self.conns:
            self.asm.update(c.recv())

    def sample(self, n):
        """Time per CG iteration of every face (n iterations each, all workers in parallel)."""
        for c in self.conns:
            c.send(n)
        t_it = {}
        for c in self.conns:
            t_it.update(c.recv())
        return t_it

    def solve_time(self, t_it):
        return max(sum(self.asm[i] + self.its[i] * t_it[i] for i in faces) for faces in self.plan)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=10)


def _cpu_baseline(config, n_it=24):
    """The oracle as it stands, bounded sample, on the host cores (rank 0, N = 1 only)."""
    pool = OraclePool(config)
    try:
        t_it = pool.sample(n_it)
        t = pool.solve_time(t_it)
    finally:
        pool.close()
    tot_it = sum(pool.its)
    unit = "full-sky solves/s" if config == "fullsky" else "solves/s"
    return {"value": 1.0 / t, "unit": unit, "cores": pool.workers, "kind": "oracle",
            "sample": (f"oracle (scipy CSR, literal Kronecker assembly, textbook HS-CG), {pool.workers} processes x 1 "
                       f"thread over the {len(pool.its)} faces of '{config}': each face assembled (timed) + {n_it} "
                       f"CG iterations (timed); extrapolated with the oracle's own iteration counts "
                       f"({tot_it} face-iterations, tests/golden/oracle_iterations.json) to the slowest worker"),
            "s_per_face_iteration_mean": statistics.mean(t_it.values()),
            "s_assembly_mean": statistics.mean(pool.asm.values()),
            "cg_iters_per_s": tot_it / t}


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
    c = CONFIGS[args.config]
    pool = OraclePool(args.config)
    vals = []
    try:
        for step in range(args.warmup + args.steps):
            t_it = pool.sample(args.ref_iters)
            if step >= args.warmup:
                vals.append(pool.solve_time(t_it))
    finally:
        pool.close()
    t_solve = statistics.mean(vals)
    val = 1.0 / t_solve
    unit = "full-sky solves/s" if args.config == "fullsky" else "solves/s"
    sample = (f"per step: {args.ref_iters} textbook CG iterations of every face on {pool.workers} oracle processes "
              f"(1 thread each; faces assembled once, timed); extrapolated to one solve = slowest worker's "
              f"sum of (assembly + oracle iterations x time per iteration), {sum(pool.its)} face-iterations")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": unit,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_solve * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/ recipe, SURVEY 8(d)); CPU fp64 oracle",
        "config": {"workload": args.config, "level": c["level"], "n": c["n"], "k": c["k"],
                   "patches": len(c["seeds"]), "tol": TOL, "route": "kron"},
        "cpu_baseline": {"value": val, "unit": unit, "cores": pool.workers, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cg_iters_per_s": sum(pool.its) / t_solve,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU legs
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
    out = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
           "unit": "full-sky solves/s" if args.config == "fullsky" else "solves/s",
           "lanczos_steps_per_face": reps[-1]["iterations_per"], "mode": "hbm-resident basis (lanczos_store)",
           "true_rel_residual": reps[-1]["rel_residual_true"],
           "roofline": roof3(reps, problems[0].k, problems[0].N, "lanczos_kernel + lz_assemble_kernel",
                             traffic_key=f"{args.config}/lanczos",
                             model_bytes=sum(r["loop_bytes"] for r in reps),
                             note="algorithmic bytes of the block-Lanczos pass structure (DESIGN.md 6); ncu "
                                  "traffic of the lanczos_kernel launch alone")}
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
    peak, _ = _peaks()
    b2 = sum(r["loop_bytes"] for r in reps2)
    tl2 = sum(r["loop_time_s"] for r in reps2)
    out["replay_mode"] = {"value": len(reps2) / t2, "ms_per_step": t2 / len(reps2) * 1e3,
                          "mode": "second Lanczos pass (P:L520-528), 4 block slots",
                          "roofline_frac": b2 / tl2 / 1e9 / peak}
    del ctx, Y, mu
    torch.cuda.empty_cache()
    return out


def _ctx_leg(problems, st, dev, timed, args, name, route="kron", traffic_key=None, kernel="cg_persistent_kernel",
             clocks_dev=None, **kw):
    """A CG-kernel leg on its own context (precond / cg_variant options): value + three-way roofline."""
    import torch
    from paper_2204_08057_b200.kroncg import KronCG
    ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev, **kw)
    Y = torch.from_numpy(st["Y"]).to(dev)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    call = {"kron": ctx.solve, "sylvester": ctx.sylvester, "kohler": ctx.kohler}[route]
    fn = lambda: call(Y, mu, tol=TOL)[1]
    for _ in range(max(1, args.warmup // 2)):
        r = fn()
        assert r["converged"], (name, r["status_name"])
    clk = ClockSampler(clocks_dev) if clocks_dev is not None else None
    t, reps = timed(fn, args.steps)
    clocks = clk.stop() if clk is not None else None
    K = problems[0].k if route == "kron" else 1
    out = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
           "unit": "full-sky solves/s" if args.config == "fullsky" else "solves/s",
           "system_iterations_per_solve": reps[-1]["system_iterations"],
           "iterations_per_system": reps[-1]["iterations_per"],
           "true_rel_residual": reps[-1]["rel_residual_true"],
           "kernel_launches_per_solve": reps[-1]["kernel_launches"],
           "roofline": roof3(reps, K, problems[0].N, kernel, traffic_key=traffic_key)}
    if clocks is not None:
        out["clocks"] = clocks
    del ctx, Y, mu
    torch.cuda.empty_cache()
    return out


def _variance_leg(ctx, timed, args, K, N, n_probes=4):
    """Posterior variances (posterior_variance: Hutchinson) on this rank's faces:
    one step = n_probes probes, each one batched CG solve of every face with b = the probe."""
    fn = lambda: ctx.posterior_variance(n_probes, seed=11, tol=TOL)[1]
    r = fn()
    assert r["status"] == 0, r["status_name"]
    t, reps = timed(fn, max(1, args.steps // 2))
    # one report per step aggregates n_probes launches: count them as launches
    rr = [dict(r, n_systems=r["n_systems"] * n_probes) for r in reps]
    roof = roof3(rr, K, N, "cg_persistent_kernel")
    roof["avg_launch_ms"] /= n_probes
    roof["algorithmic_bytes_per_launch"] /= n_probes
    roof["bytes_moved"]["per_launch"] /= n_probes
    tr = _traffic(f"{args.config}/variance")  # DRAM bytes of one probe solve's CG launch (ncu)
    if tr:
        tl = roof["avg_launch_ms"] * 1e-3
        roof["traffic"] = tr
        roof["ncu_dram"] = {"per_launch": tr, "achieved": tr / tl / 1e9, "frac": tr / tl / 1e9 / roof["peak"],
                            "source": f"profiles/ncu_traffic.json[{args.config}/variance]"}
    return {"value": len(reps) * n_probes / t, "unit": "probe solves/s (all faces of the rank per probe)",
            "probes_per_step": n_probes, "ms_per_step": t / len(reps) * 1e3,
            "face_iterations_per_probe": reps[-1]["system_iterations"] / n_probes,
            "roofline": roof}


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
    k, N = ps[0].k, ps[0].N
    for name, fn in (("kron", ctx.solve), ("sylvester", ctx.sylvester), ("lanczos", ctx.lanczos)):
        call = lambda: fn(Y, mu, tol=TOL)[1]
        r = call()
        assert r["converged"], (name, r["status_name"])
        t, reps = timed(call, args.steps)
        out[name] = {"value": len(reps) / t, "ms_per_step": t / len(reps) * 1e3,
                     "iterations_per_system": reps[-1]["iterations_per"],
                     "true_rel_residual": reps[-1]["rel_residual_true"]}
        if name != "lanczos":
            out[name]["roofline"] = roof3(reps, k if name == "kron" else 1, N, "cg_march_kernel (D2 row march)",
                                          traffic_key=f"paper/{name}")
    del ctx, Y, mu, hits
    torch.cuda.empty_cache()
    return out


def _small_leg(dev, timed, args, clocks_dev):
    """The small-problem regime (tiny and medium configs, CG state resident in shared memory,
    kcg_res.cuh): solves/s and us per iteration, next to the streaming kernel on the same input."""
    import torch
    from synth import make_config
    from synth.problems import stack
    from paper_2204_08057_b200.kroncg import KronCG
    out = {}
    for cfg in ("tiny", "medium"):
        ps = make_config(cfg)
        st = stack(ps)
        Y = torch.from_numpy(st["Y"]).to(dev)
        leg = {}
        # default = the planner's choice (single-CTA resident kernel for tiny faces, the streaming
        # kernel otherwise); "streaming" forces the latter, "strips" the opt-in row-strip resident mode
        modes = {"default": None, "streaming": "0"}
        if cfg == "medium":
            modes["strips"] = "2"
        for mode, env in modes.items():
            if env is not None:
                os.environ["KCG_RESIDENT"] = env
            try:
                ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev)
            finally:
                os.environ.pop("KCG_RESIDENT", None)
            fn = lambda: ctx.solve(Y, tol=TOL)[1]
            for _ in range(max(3, args.warmup)):
                fn()
            steps = max(args.steps, 20)
            clk = ClockSampler(clocks_dev)
            t, reps = timed(fn, steps)
            clocks = clk.stop()
            it = reps[-1]["iterations"]
            lt = sum(r["loop_time_s"] for r in reps) / len(reps)
            res = ctx.launch_config()["resident_kron"] > 0
            leg[mode] = {"value": len(reps) / t, "unit": "solves/s", "ms_per_step": t / len(reps) * 1e3,
                         "iterations": it, "us_per_iteration": lt / (it + 1) * 1e6,
                         "strips_per_face": ctx.launch_config()["resident_kron"],
                         "roofline": roof3(reps, ps[0].k, ps[0].N,
                                           "cg_resident_kernel" if res else "cg_persistent_kernel",
                                           bound="latency" if res else "hbm",
                                           note=("frac = iteration rate against the streaming algorithm's HBM "
                                                 "roofline (48 K N B per pass); the resident kernel keeps x, r, p "
                                                 "in shared memory, bytes_moved = its global (L2) traffic")
                                           if res else None),
                         "clocks": clocks}
            del ctx
        leg["config"] = {"workload": cfg, "level": ps[0].level, "k": ps[0].k, "patches": len(ps)}
        out[cfg] = leg
        del Y
    torch.cuda.empty_cache()
    return out


def _planck_leg(dev, timed, args, clocks_dev):
    """The planck face alone (BASELINE configs[2]: L = 10, k = 4): the north star's >= 70 % config."""
    from synth import make_config
    from synth.problems import stack
    ps = make_config("planck")
    st = stack(ps)
    a = argparse.Namespace(**vars(args))
    a.config = "planck"
    out = _ctx_leg(ps, st, dev, timed, a, "planck", traffic_key="planck/kron", clocks_dev=clocks_dev)
    out["config"] = {"workload": "planck", "level": 10, "k": 4, "patches": 1}
    out["us_per_iteration"] = out["roofline"]["avg_launch_ms"] * 1e3 / (out["system_iterations_per_solve"] + 1)
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    world, rank, local = _dist()
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # more ranks than GPUs (the multi-process test of the face-shard path, KCG_BENCH_BACKEND=gloo):
    # ranks share devices round-robin; nothing on this path waits on another rank's kernels
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("KCG_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # several ranks on one GPU (multi-process tests): gloo for the host-side barrier / max
            dist.init_process_group(backend)
    cpu_coll = backend != "nccl"

    from paper_2204_08057_b200 import build
    if rank == 0 or world == 1:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2204_08057_b200.kroncg import KronCG
    from synth.problems import stack

    from synth import CONFIGS
    whole = args.shard_only or (not args.row_slabs and len(CONFIGS[args.config]["seeds"]) >= world)
    problems, mine, costs, g, slab = _patches_for(args.config, world, rank, whole)
    st = stack(problems)
    K, N = problems[0].k, problems[0].N
    if g == 1:
        ctx = KronCG(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                     device=dev, host_staging=2)
        Yn = st["Y"]
    else:
        # every rank creates every group (same order), then joins its own: slabs of its group's faces
        from paper_2204_08057_b200.kroncg import KronCGSlab, split_rows
        groups = [dist.new_group(list(range(j * g, (j + 1) * g))) for j in range(world // g)]
        ctx = KronCGSlab(problems[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], g,
                         emulate=False, group=groups[rank // g], device=dev, host_staging=True)
        Yn = split_rows(st["Y"], g)[slab:slab + 1]
        N = N // g
    Y = torch.from_numpy(Yn).to(dev)
    mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
    Y_host = torch.from_numpy(Yn).pin_memory()
    mu_host = [torch.empty(mu.shape, dtype=torch.float64).pin_memory() for _ in range(2)]
    stream = torch.cuda.current_stream(dev)

    def allmax(v):
        if world == 1:
            return v
        tt = torch.tensor([v], dtype=torch.float64, device="cpu" if cpu_coll else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

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
        return allmax(e0.elapsed_time(e1) / 1e3), reps

    kron = lambda: ctx.solve(Y, mu, tol=TOL)[1]
    syl = lambda: ctx.sylvester(Y, mu, tol=TOL)[1]
    main_fn = kron if args.route == "kron" else syl
    other_fn = syl if args.route == "kron" else kron

    for _ in range(args.warmup):
        r = main_fn()
        assert r["converged"], r
    clk = ClockSampler(local)
    t_main, reps = timed(main_fn, args.steps)
    clocks = clk.stop()
    # this rank's own busy time of the main leg (the max over ranks is t_main): per-GPU busy time and
    # the sharding's makespan bound go into the line for N > 1
    t_busy_local = sum(r["loop_time_s"] for r in reps)
    for _ in range(max(1, args.warmup // 2)):
        other_fn()
    t_other, reps_other = timed(other_fn, args.steps)
    # e2e: the pipelined host entry point (g == 1) or the blocking one (slab ranks), every step's
    # H2D of Y and D2H of mu inside the timed region
    n_e2e = max(2, args.e2e_steps)
    if g == 1:
        host = lambda: ctx.solve_host_many([Y_host] * n_e2e, [mu_host[i & 1] for i in range(n_e2e)], tol=TOL)
        host()
        t_e2e, reps_e2e = timed(host, 1)
        e2e_api = "kron_cg_solve_host_many (C ABI, pinned host buffers, copies overlapped with the solves)"
    else:
        host = lambda: ctx.solve_host(Y_host, mu_host[0], tol=TOL)[1]
        host()
        t_e2e, reps_e2e = timed(host, n_e2e)
        e2e_api = "kron_cg_solve_host (C ABI, pinned host buffers)"
    extra = {}
    if g == 1 and not args.no_lanczos:
        extra["lanczos"] = _lanczos_leg(problems, st, dev, timed, args, cpu=(world == 1))
    if g == 1 and not args.no_hs:
        extra["hs_variant"] = _ctx_leg(problems, st, dev, timed, args, "hs", traffic_key=f"{args.config}/hs",
                                       kernel="cg_hs_kernel", cg_variant="hs")
        extra["hs_variant"]["note"] = ("textbook Hestenes-Stiefel CG (Alg. CG P:L225-241, two grid reductions, "
                                       "72 K N B per iteration; reading R9) -- the single-pass kernel's baseline")
    if g == 1 and not args.no_pcg:
        extra["pcg_block_jacobi"] = _ctx_leg(problems, st, dev, timed, args, "pcg", traffic_key=f"{args.config}/pcg",
                                             kernel="cg_persistent_kernel (PREC)", precond="block_jacobi")
    if g == 1 and not args.no_kohler:  # Alg. Kohler (NEXT-4): k sequential batched column solves
        call = lambda: ctx.kohler(Y, mu, tol=TOL)[1]
        rk = call()
        assert rk["converged"], rk["status_name"]
        tk, reps_k = timed(call, args.steps)
        extra["kohler"] = {"value": len(reps_k) / tk, "ms_per_step": tk / len(reps_k) * 1e3,
                           "system_iterations_per_solve": reps_k[-1]["system_iterations"],
                           "roofline": roof3(reps_k, 1, N, "cg_persistent_kernel (K = 1, one launch per column) "
                                             "+ column kernels", traffic_key=f"{args.config}/kohler")}
    if g == 1 and not args.no_variance:
        extra["posterior_variance"] = _variance_leg(ctx, timed, args, K, N)
    if world == 1 and not args.no_paper:
        extra["paper_workload"] = _paper_leg(dev, timed, args)
    if world == 1 and not args.no_planck and args.config != "planck":
        extra["planck"] = _planck_leg(dev, timed, args, local)
    if world == 1 and not args.no_small:
        extra["small"] = _small_leg(dev, timed, args, local)

    def agg(reps_):
        loc = [sum(r["system_iterations"] for r in reps_), sum(r["kernel_launches"] for r in reps_),
               1.0 if slab == 0 else 0.0]
        if world == 1:
            return [loc]
        t = torch.tensor(loc, dtype=torch.float64, device="cpu" if cpu_coll else dev)
        allv = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allv, t)
        return [v.tolist() for v in allv]

    g_main = agg(reps)
    g_other = agg(reps_other)
    if world > 1:
        tb = torch.tensor([t_busy_local, float(sum(costs[i] for i in mine)) / g], dtype=torch.float64,
                          device="cpu" if cpu_coll else dev)
        tbs = [torch.zeros_like(tb) for _ in range(world)]
        dist.all_gather(tbs, tb)
        busy = [float(v[0].item()) for v in tbs]
        load = [float(v[1].item()) for v in tbs]
    io = torch.tensor([float(Y_host.numel() * 8), float(mu_host[0].numel() * 8)], dtype=torch.float64,
                      device="cpu" if cpu_coll else dev)
    if world > 1:
        dist.all_reduce(io)  # whole-job bytes moved by the e2e step (every rank's own slab / faces)
    h2d_bytes, d2h_bytes = int(io[0].item()), int(io[1].item())
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    S = args.steps
    unit = "full-sky solves/s" if args.config == "fullsky" else "solves/s"
    sys_its_main = sum(v[0] for v in g_main if v[2] > 0) / S  # each group's faces counted once
    launches = int(sum(v[1] for v in g_main))
    line = {
        "metric": METRIC,
        "value": S / t_main,
        "unit": unit,
        "n_gpus": world, "steps": S, "warmup": args.warmup,
        "ms_per_step": t_main / S * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth/ recipe of SURVEY 8(d), seeds per BASELINE config)",
        "config": {"workload": args.config, "level": problems[0].level, "n": problems[0].n,
                   "k": problems[0].k, "patches": len(costs), "tol": TOL, "route": args.route,
                   "parallelism": f"face-shard{world}" if g == 1 else f"face-groups{world // g}x-rowslab{g}",
                   "l2": "no flush: inputs (Y) and solver state exceed the 126 MB L2"},
        "cg_iters_per_s": sys_its_main * S / t_main,
        "face_iterations_per_solve": sys_its_main,
        "iterations_per_face_rank0": reps[-1]["iterations_per"],
        "roofline": roof3(reps, K if args.route == "kron" else 1, N, "cg_persistent_kernel",
                          traffic_key=f"{args.config}/{args.route}"),
        "e2e": {"value": (n_e2e if g == 1 else len(reps_e2e)) / t_e2e, "unit": unit,
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes, "api": e2e_api,
                "steps": n_e2e},
        # counted by the library at each of its kernel launches (report.kernel_launches), all ranks
        "gpu_launches": launches,
        "gpu_launches_per_step_rank0": reps[-1]["kernel_launches"],
        "clocks": clocks,
        "sylvester" if args.route == "kron" else "kron": {
            "value": S / t_other, "ms_per_step": t_other / S * 1e3,
            "system_iterations_per_solve": sum(v[0] for v in g_other if v[2] > 0) / S,
            "roofline": roof3(reps_other, 1 if args.route == "kron" else K, N, "cg_persistent_kernel",
                              traffic_key=f"{args.config}/{'sylvester' if args.route == 'kron' else 'kron'}")},
        "true_rel_residual": reps[-1]["rel_residual_true"],
    }
    line.update(extra)
    if world > 1:  # per-GPU busy time of the CG loop (all steps) next to the cost model's makespan bound
        line["sharding"] = {
            "faces_per_group": len(mine), "group_size": g,
            "cg_loop_busy_s_per_rank": busy,
            "modelled_load_per_rank": load,
            "modelled_speedup_bound": sum(costs) / max(max(load), 1e-30),
            "note": "load = the sqrt(cond) cost of the faces a rank's group holds / g (row slabs); bound = "
                    "total cost / the largest rank load (the cost model's makespan, exchange not counted)"}
    if world == 1 and not args.no_slab_probe:
        line["slab_emulation"] = _slab_probe(dev)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(args.config)
        if "posterior_variance" in line:  # the oracle's Hutchinson probe = one oracle CG solve per face
            cb = line["cpu_baseline"]
            var = line["posterior_variance"]
            t_probe = len(problems) * cb["s_assembly_mean"] / cb["cores"] + \
                var["face_iterations_per_probe"] * cb["s_per_face_iteration_mean"] / cb["cores"]
            var["cpu_baseline"] = {"value": 1.0 / t_probe, "unit": var["unit"], "cores": cb["cores"], "kind": "oracle",
                                   "sample": "oracle.variance.hutchinson = oracle.cg.cg_hs per probe and face; "
                                             "timed by the Kron-CG sample above (same CG, same operator, same pool)"}
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
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-slab-probe", action="store_true")
    ap.add_argument("--no-lanczos", action="store_true", help="skip the block-Lanczos (Alg. SylvSolver) leg")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper-workload leg (App. B physics, D^2)")
    ap.add_argument("--no-variance", action="store_true", help="skip the posterior-variance (Hutchinson) leg")
    ap.add_argument("--no-pcg", action="store_true", help="skip the block-Jacobi preconditioned CG leg")
    ap.add_argument("--no-kohler", action="store_true", help="skip the Alg. Kohler leg")
    ap.add_argument("--no-hs", action="store_true", help="skip the textbook HS CG variant leg")
    ap.add_argument("--no-planck", action="store_true", help="skip the planck-face leg")
    ap.add_argument("--no-small", action="store_true", help="skip the tiny / medium (resident kernel) legs")
    ap.add_argument("--shard-only", action="store_true",
                    help="N > 1: whole faces per rank only (no row-slab groups), e.g. several ranks on one GPU")
    ap.add_argument("--row-slabs", action="store_true",
                    help="N > 1 with at least as many faces as ranks: let the planner split faces into row slabs "
                         "(sharding.plan_groups).  Off by default: the cross-GPU slab solve (kernels spinning on "
                         "each other's flags over NVLink) cannot run on this one-GPU pool, and on fullsky the model "
                         "gains 2%% at 8 ranks (32.2 vs 32.9 face-passes).  Single-face configs always use slabs")
    ap.add_argument("--lanczos-cap", type=int, default=128,
                    help="Lanczos steps provisioned (HBM-resident basis: P k N 8 (cap + 1) bytes)")
    ap.add_argument("--ref-iters", type=int, default=2, help="oracle CG iterations per face per reference step")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        print("warning: warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
