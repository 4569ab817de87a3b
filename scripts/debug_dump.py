"""Debug helper (KCG_TRACE=2 build): smem snapshots of the first tile of the start pass."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_patch
from synth.problems import stack
from oracle import cg, model
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
for k, prec in [(2, "block_jacobi"), (2, "none")]:
    p = make_patch(3, 9, k, seed=1, tau="loguniform")
    st = stack([p])
    Y = torch.from_numpy(st["Y"]).cuda()
    ctx = KronCG(3, st["A"], st["noise_prec"], st["tau"], st["kappa2"], precond=prec)
    mu, rep = ctx.solve(Y, tol=1e-10, max_iter=0, allow=tuple(range(10)))
    buf = np.zeros(1024 * 160, dtype=np.int64)
    f(ctx._ctx, buf.ctypes.data, 1024)
    d = buf.view(np.float64)
    TY, BW, BH = 16, 68, 20
    PLANE = BW * BH
    G, b = model.problem_system(p)
    B = b.reshape(k, 8, 8)
    exp = np.zeros((k, BH, BW)); exp[:, 2:10, 2:10] = B
    for sec, name in [(0, "R@tma"), (1, "R@B"), (2, "R@B'")]:
        R = d[sec * 8192: sec * 8192 + k * PLANE].reshape(k, BH, BW)
        diff = np.abs(R - exp)
        print(prec, name, "max diff", diff.max(), "where", np.argwhere(diff > 1e-9)[:8].tolist(), flush=True)
    if prec != "none":
        UPLANE = BW * (TY + 2)
        U = d[3 * 8192: 3 * 8192 + k * UPLANE].reshape(k, TY + 2, BW)
        K = cg.block_jacobi_precond(3, p.A, p.noise_prec, p.tau, p.kappa2)
        u = K(b).reshape(k, 8, 8)
        uexp = np.zeros((k, TY + 2, BW)); uexp[:, 1:9, 2:10] = u
        diff = np.abs(U - uexp)
        print("U max diff", diff.max(), "n bad", int((diff > 1e-9).sum()), np.argwhere(diff > 1e-9)[:20].tolist())
        print("U region rows 0..9 cols 0..12 plane 0:\n", np.round(U[0, :10, :12], 2))
        print("U expected:\n", np.round(uexp[0, :10, :12], 2))
    tred = d[4 * 8192: 4 * 8192 + 3 * 16].reshape(3, 16)
    print("tred sums", tred.sum(1), "b.b", b @ b, flush=True)
    print("tred rr per warp", tred[0], "\nexpected", (B ** 2).sum(axis=(0, 2)))
    th = d[5 * 8192: 5 * 8192 + 512 * k * 8].reshape(512, k, 8)
    for tid in list(range(128, 132)) + list(range(160, 164)):
        print("tid", tid, np.round(th[tid], 3).tolist())
    print("expected row4", B[:, 4, :4], "row5", B[:, 5, :4])
