"""Paper workload (App. B physics, D^2, hits, NESTED; 12 faces, L = 10): loop time of the Kronecker-CG
and Sylvester routes (row-march kernels), best of 3 after a warm-up.  usage: paper_routes_probe.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth.physics import make_paper_patch, nested_order
from synth.problems import stack
ps = [make_paper_patch(10, seed=400 + f) for f in range(12)]
st = stack(ps)
ctx = KronCG(10, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=torch.from_numpy(nested_order(st["hits"])).cuda(),
             layout="nested", prior="d2")
Y = torch.from_numpy(nested_order(st["Y"])).cuda()
for route, fn in (("kron", ctx.solve), ("sylvester", ctx.sylvester)):
    ts = []
    for _ in range(4):
        mu, r = fn(Y, tol=1e-10)
        ts.append(r["loop_time_s"] * 1e3)
    its = r["system_iterations"]
    print(json.dumps(dict(route=route, loop_ms=round(min(ts[1:]), 3), wall_ms=round(r["wall_time_s"] * 1e3, 3),
                          us_per_system_iter=round(min(ts[1:]) * 1e3 / max(its, 1), 2),
                          loop_GBs=round(r["loop_bytes"] / (min(ts[1:]) * 1e-3) / 1e9, 1),
                          rel_true=r["rel_residual_true"], its=r["iterations_per"][:4])))
