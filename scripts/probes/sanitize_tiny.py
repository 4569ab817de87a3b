"""Tiny solves through every route (for compute-sanitizer): Kron CG (streaming tile kernel and the
resident kernel), Sylvester, block Lanczos, Kohler, block-Jacobi PCG, D2 row march, HS variant."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_patch
from synth.problems import stack

ps = [make_patch(6, 9, 3, seed=5 + s, tau="loguniform", hits="random") for s in range(2)]
st = stack(ps)
h = torch.from_numpy(st["hits"]).cuda()
Y = torch.from_numpy(st["Y"]).cuda()
for kw in ({}, {"precond": "block_jacobi"}, {"prior": "d2"}, {"cg_variant": "hs"}, {"lanczos_cap": 64}):
    ctx = KronCG(6, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=h, **kw)
    _, r = ctx.solve(Y, tol=1e-10)
    print(kw, "kron", r["iterations_per"], r["status_name"])
    if not kw or "lanczos_cap" in kw:
        _, r = ctx.sylvester(Y, tol=1e-10)
        print(kw, "sylvester", r["iterations_per"], r["status_name"])
        _, r = ctx.kohler(Y, tol=1e-10)
        print(kw, "kohler", r["iterations_per"], r["status_name"])
    if "lanczos_cap" in kw:
        _, r = ctx.lanczos(Y, tol=1e-10)
        print(kw, "lanczos", r["iterations_per"], r["status_name"])
torch.cuda.synchronize()
print("done")
