"""Paper workload (App. B physics, D^2 with kappa2 = 0, hits, NESTED): how close is the GPU Kron-CG
iterate to the oracle's HS-CG and single-pass iterates, and how close are the oracle's two variants to
each other and to the direct solve?  Prints one line per face (sizes the parity tolerance)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import scipy.sparse.linalg as ssl
import torch
from oracle import cg, model
from synth.physics import make_paper_patch
from synth.problems import stack
from paper_2204_08057_b200.kroncg import KronCG


def rel(a, b):
    a, b = np.ravel(a), np.ravel(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


for level in (5, 6, 7):
    ps = [make_paper_patch(level, seed=200 + s) for s in range(3)]
    st = stack(ps)
    nest = lambda a: model.to_layout(level, a, "nested").reshape(np.shape(a))
    ctx = KronCG(level, st["A"], st["noise_prec"], st["tau"], st["kappa2"],
                 hits=torch.from_numpy(nest(st["hits"])).cuda(), layout="nested", prior="d2")
    Y = torch.from_numpy(nest(st["Y"])).cuda()
    mu, rep = ctx.solve(Y, tol=1e-10)
    mu = mu.cpu().numpy()
    for i, p in enumerate(ps):
        G, b = model.problem_system(p, layout="nested")
        ref = ssl.spsolve(G.tocsc(), b)
        o = cg.cg_hs(G, b, tol=1e-10)
        sp = cg.cg_single_pass(G, b, tol=1e-10)
        ev = ssl.eigsh(G, k=1, which="LA", return_eigenvectors=False)[0]
        evm = ssl.eigsh(G, k=1, sigma=0, which="LM", return_eigenvectors=False)[0]
        x = mu[i].reshape(-1)
        print(f"L={level} face {i}: it gpu {rep['iterations_per'][i]} hs {o.iterations} sp {sp.iterations} | "
              f"rel(gpu,hs) {rel(x, o.x):.2e} rel(gpu,sp) {rel(x, sp.x):.2e} rel(hs,sp) {rel(o.x, sp.x):.2e} | "
              f"rel(gpu,ref) {rel(x, ref):.2e} rel(hs,ref) {rel(o.x, ref):.2e} cond {ev / evm:.2e}", flush=True)
