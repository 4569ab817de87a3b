"""Time the Kronecker-CG and Sylvester routes with the D^2 prior (the paper's operator) on a config:
usage: d2_cg_probe.py CONFIG [paper]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack

name = sys.argv[1] if len(sys.argv) > 1 else "planck"
ps = make_config(name, prior="d2")
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], prior="d2")
Y = torch.from_numpy(st["Y"]).cuda()
for route, fn in (("kron", ctx.solve), ("sylvester", ctx.sylvester)):
    for _ in range(3):
        mu, r = fn(Y, tol=1e-10)
    its = r["system_iterations"]
    print(json.dumps(dict(config=name, route=route, prior="d2", iterations=r["iterations_per"][:12],
                          loop_ms=r["loop_time_s"] * 1e3, us_per_system_iter=r["loop_time_s"] * 1e6 / max(its, 1),
                          loop_GBs=r["loop_bytes"] / r["loop_time_s"] / 1e9, rel_true=r["rel_residual_true"])))
