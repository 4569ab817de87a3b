"""One D^2 solve on a config and route (for ncu captures of the row-march kernel):
usage: d2_one.py CONFIG ROUTE [iters]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack

name = sys.argv[1] if len(sys.argv) > 1 else "planck"
route = sys.argv[2] if len(sys.argv) > 2 else "kron"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 40
ps = make_config(name, prior="d2")
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], prior="d2")
Y = torch.from_numpy(st["Y"]).cuda()
fn = ctx.solve if route == "kron" else ctx.sylvester
mu, r = fn(Y, tol=1e-300, max_iter=iters)
print(name, route, r["loop_time_s"] * 1e6 / (iters + 1), "us per pass")
