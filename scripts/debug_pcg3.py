"""Debug helper: start-pass scalars of block-Jacobi PCG vs the oracle (GPU)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from synth import make_patch
from synth.problems import stack
from oracle import cg, model
from paper_2204_08057_b200 import build
build.build()
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG
f = kroncg._lib.kcg_debug_state
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
for level, k, hits in [(3, 2, None), (3, 3, None)]:
    p = make_patch(level, 9, k, seed=1, tau="loguniform")
    st = stack([p])
    Y = torch.from_numpy(st["Y"]).cuda()
    h = torch.ones((1, p.side, p.side), dtype=torch.float64, device="cuda") if hits else None
    ctx = KronCG(level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], hits=h, precond="block_jacobi")
    G, b = model.problem_system(p)
    K = cg.block_jacobi_precond(level, p.A, p.noise_prec, p.tau, p.kappa2)
    u = K(b); w = G @ u
    print(level, k, hits, "oracle bb", b @ b, "gamma", b @ u, "delta", w @ u, "alpha0", (b @ u) / (w @ u))
    for mi in (0, 1):
        mu, rep = ctx.solve(Y, tol=1e-10, max_iter=mi, allow=tuple(range(10)))
        out = np.zeros(9)
        f(ctx._ctx, out.ctypes.data, 1)
        print("   gpu mi", mi, "bnorm2", out[0], "gamma", out[1], "alpha", out[2], "beta", out[3], "rel", out[4], "alpha_last", out[8])
    # oracle first iteration
    r1 = b - (b @ u) / (w @ u) * (G @ u)
    u1 = K(r1); w1 = G @ u1
    g1 = r1 @ u1; d1 = w1 @ u1; beta = g1 / (b @ u); a1 = g1 / (d1 - beta * g1 / ((b @ u) / (w @ u)))
    print("   oracle it1 gamma", g1, "delta", d1, "beta", beta, "alpha1", a1, "rel", np.linalg.norm(r1) / np.linalg.norm(b))
print(ctx.launch_config())
