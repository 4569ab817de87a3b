"""Paper workload (App. B physics, D^2, hits, NESTED; 12 faces, L = 10): one Kronecker-CG solve (for an
ncu capture of the D2 row-march kernel)."""
import os, sys
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
mu, r = ctx.solve(Y, tol=1e-10)
print(r["iterations_per"], r["loop_time_s"] * 1e3)
