"""One warm-up solve, then ONE profiled solve (cudaProfilerStart/Stop range, for
`ncu --profile-from-start off`) of a config and route.  usage: solve_once.py CONFIG ROUTE
(CONFIG: a synth config or "paper" = App. B physics, D2, hits, NESTED; ROUTE: kron, sylvester, kohler,
hs, pcg, lanczos, variance)"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth.problems import stack

cfg, route = sys.argv[1], sys.argv[2]
kw = {}
if route == "hs":
    kw["cg_variant"] = "hs"
if route == "pcg":
    kw["precond"] = "block_jacobi"
if route == "lanczos":
    kw["lanczos_cap"] = 128
    kw["lanczos_store"] = True
if cfg == "paper":
    from synth.physics import make_paper_patch, nested_order
    ps = [make_paper_patch(10, seed=400 + f) for f in range(12)]
    st = stack(ps)
    ctx = KronCG(10, st["A"], st["noise_prec"], st["tau"], st["kappa2"], layout="nested", prior="d2",
                 hits=torch.from_numpy(nested_order(st["hits"])).cuda(), **kw)
    Y = torch.from_numpy(nested_order(st["Y"])).cuda()
else:
    from synth import make_config
    ps = make_config(cfg)
    st = stack(ps)
    ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], **kw)
    Y = torch.from_numpy(st["Y"]).cuda()
fn = {"kron": ctx.solve, "hs": ctx.solve, "pcg": ctx.solve, "sylvester": ctx.sylvester, "kohler": ctx.kohler,
      "lanczos": ctx.lanczos, "variance": lambda Y, tol: ctx.posterior_variance(1, seed=1, tol=tol)}[route]
fn(Y, tol=1e-10)
torch.cuda.synchronize()
torch.cuda.profiler.start()
_, rep = fn(Y, tol=1e-10)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, route, rep.get("system_iterations"), rep.get("loop_time_s"), rep.get("loop_bytes"))
