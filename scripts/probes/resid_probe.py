"""fullsky: 2 Kron solves + 2 Sylvester solves (the residual apply kernel runs once per solve), for ncu."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack
ps = make_config("fullsky")
st = stack(ps)
ctx = KronCG(10, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
for _ in range(2):
    ctx.sylvester(Y, tol=1e-10)
